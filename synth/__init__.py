"""Seeded synthetic INPUT generators shared by the oracle side and the CUDA side.

This package holds none of the method's arithmetic (no CNN, pyramid, patch,
equalisation, decision rule or grouping code).  It produces only inputs:

* ``arch``    -- the layer lists of the reconstructed architecture R (SURVEY.md §8,
                 "Reconstructed architecture R"); an input to ``ccnn_create`` and to
                 the oracle alike.
* ``weights`` -- random-init weights (splitmix64, LeCun-uniform), DESIGN.md "Inputs".
* ``frames``  -- integer-only hash-lattice value-noise frames with planted face
                 templates, video streams and clutter.
* ``configs`` -- the five BASELINE.json workloads C1..C5 as plain parameter records.
"""

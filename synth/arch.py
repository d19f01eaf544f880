"""Layer lists of the reconstructed architecture R (an input, not method arithmetic).

PAPER.md Fig. 1 is missing from the extracted text.  What the text fixes:
conv stride 1, pool stride 2, no fully-connected layer (§3.1); CNN1 scans a
27x31 window at a 4-px step (§3.3); CNN2/CNN3 map a 51x55 patch to a 5x5
response map; the nets have 797, 1,819 and 2,923 parameters.
R is the unique fully-connected, untrainable-pool solution
with a final 1x1 conv that meets all of these; DESIGN.md "Readings" R1.

A layer is ``(kind, in_maps, out_maps, kw, kh)``:
kind 0 = valid conv (stride 1, bias) followed by the Eq. 1 activation,
kind 1 = 2x2 max-pool, stride 2, floor.  Kernel sizes are width x height.
"""

CONV, POOL = 0, 1

CNN1 = (
    (CONV, 1, 6, 4, 4),
    (POOL, 6, 6, 2, 2),
    (CONV, 6, 6, 3, 3),
    (POOL, 6, 6, 2, 2),
    (CONV, 6, 2, 5, 6),
    (CONV, 2, 1, 1, 1),
)

CNN2 = (
    (CONV, 1, 16, 4, 4),
    (POOL, 16, 16, 2, 2),
    (CONV, 16, 6, 3, 3),
    (POOL, 6, 6, 2, 2),
    (CONV, 6, 2, 7, 8),
    (CONV, 2, 1, 1, 1),
)

CNN3 = (
    (CONV, 1, 2, 4, 4),
    (POOL, 2, 2, 2, 2),
    (CONV, 2, 2, 3, 3),
    (POOL, 2, 2, 2, 2),
    (CONV, 2, 25, 7, 8),
    (CONV, 25, 1, 1, 1),
)

NETS = (CNN1, CNN2, CNN3)

# Paper's parameter counts (§3.1) -- used by tests as the pin, not derived here.
PAPER_PARAM_COUNTS = (797, 1819, 2923)

# Stage-1 window and selective patch / response map.
WINDOW_W, WINDOW_H = 27, 31
PATCH_W, PATCH_H = 51, 55
RESP_W, RESP_H = 5, 5

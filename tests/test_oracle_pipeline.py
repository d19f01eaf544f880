"""Pins for the oracle's end-to-end detect (Fig. 3; SPEC detect S:338-350).

Invariants: all windows survive below the activation range, candidate sets
shrink monotonically in T1, Table-1 stage counts are non-increasing under
Eq. 2, dense scan == per-window definition end to end, and the
stats' window count equals the closed-form grid sum.
"""
import numpy as np

import oracle
from synth import frames

RNG = np.random.default_rng(3)


def _small_frame(seed=11, W=72, H=64):
    return frames.make_still(W, H, seed, 27)


def test_all_windows_survive_below_range(cascade):
    f = _small_frame()
    cands, boxes, st = oracle.detect(cascade, f, 27, 1.25, -1.75, (0.0, 0.0), 2, 0)
    lv = oracle.level_table(f.shape[1], f.shape[0], 27, 1.25)
    total = sum(oracle.window_grid(lw, lh)[0] * oracle.window_grid(lw, lh)[1] for _, lw, lh in lv)
    assert st["windows"] == total == len(cands) == st["stage1"]
    # every (level, i, j) exactly once
    keys = {(c["level"], c["iy"], c["ix"]) for c in cands}
    assert len(keys) == total


def test_t1_monotone_and_stage_counts(cascade):
    f = frames.make_still(160, 120, 21, 24)
    prev = None
    for T1 in (-0.5, -0.1, 0.05, 0.2, 0.4):
        cands, boxes, st = oracle.detect(cascade, f, 24, 1.2, T1, (0.1, 0.1), 2, 0)
        keys = {(int(c["level"]), int(c["iy"]), int(c["ix"])) for c in cands}
        if prev is not None:
            assert keys <= prev
        prev = keys
        assert st["windows"] >= st["stage1"] >= st["stage2"] >= st["stage3"] >= st["nms"]
        assert all(c["s1"] > T1 or np.float32(c["s1"]) > np.float32(T1) for c in cands)


def test_dense_equals_per_window_detect(cascade):
    f = frames.make_still(120, 100, 8, 24)
    a = oracle.detect(cascade, f, 24, 1.2, 0.1, (0.05, 0.05), 2, 0, dense=True)
    b = oracle.detect(cascade, f, 24, 1.2, 0.1, (0.05, 0.05), 2, 0, dense=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_weak_rule_and_thread_determinism(cascade):
    f = np.stack([_small_frame(1), _small_frame(2)])
    a = oracle.detect(cascade, f, 27, 1.2, 0.0, (0.0, 0.0), 2, 1, n_threads=1)
    b = oracle.detect(cascade, f, 27, 1.2, 0.0, (0.0, 0.0), 2, 1, n_threads=8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    cands = a[0]
    for c in cands:
        if c["K2"] >= 2:
            assert c["delta"] == 1 and c["cnn3_ran"] == 0          # Eq. 3 short-cut
    assert set(np.unique(cands["frame"])) <= {0, 1}


def test_empty_pyramid_is_not_an_error(cascade):
    f = np.zeros((20, 20), np.uint8)
    cands, boxes, st = oracle.detect(cascade, f, 27, 1.2, 0.0, (0.0, 0.0), 2, 0)
    assert len(cands) == 0 and len(boxes) == 0 and st["windows"] == 0

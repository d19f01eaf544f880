"""CPU checks of the parity harness itself (tests/parity.py), no GPU.

The GPU parity tests are only as strong as the comparison code, so it is exercised here on
"GPU outputs" built from the oracle's own results (which must pass) and on perturbed copies
(which must fail): a moved box, a dropped accepted candidate, a flipped decision, a wrong
count.  Also: threshold placement keeps a > 1e-4 margin on the frames it is placed on.
"""
import numpy as np
import pytest

import oracle
from synth import configs, frames as synth_frames

from . import parity


def _as_gpu(ocands, oboxes, ostats):
    """oracle.detect results in the ABI's record types (float32 scores / responses)."""
    from paper_1508_01292_b200.ccnn import BOX_DTYPE, CAND_DTYPE
    gc = np.zeros(len(ocands), CAND_DTYPE)
    for f in CAND_DTYPE.names:
        gc[f] = ocands[f]
    gb = np.zeros(len(oboxes), BOX_DTYPE)
    for f in BOX_DTYPE.names:
        gb[f] = oboxes[f]
    return gc, gb, dict(ostats)


@pytest.fixture(scope="module")
def case(cascade):
    fr = synth_frames.make_stills(2, 333, 257, 991, 20)
    T1, T2, margins = parity.exact_thresholds(cascade, fr, 20, 1.1, 0.99, Tnn=1)
    oc, ob, st = oracle.detect(cascade, fr, 20, 1.1, T1, T2, 1, 0)
    lv = oracle.level_table(fr.shape[2], fr.shape[1], 20, 1.1)
    return fr, T1, T2, margins, oc, ob, st, [lv] * len(fr)


def _check(cascade, case, gc, gb, gst):
    fr, T1, T2, _, oc, ob, st, lvs = case
    ex = parity.exempt_windows(cascade, fr, lvs, T1)
    rep = parity.check_selective_and_boxes(gc, gb, gst, oc, ob, st, ex, fr, lvs, cascade, T1,
                                           T2, 1, 0)
    parity.check_nms(gc, gb, len(fr))
    return rep


def test_margins(case):
    assert all(m > parity.TOL for m in case[3]), case[3]


def test_oracle_output_passes(cascade, case):
    gc, gb, gst = _as_gpu(*case[4:7])
    assert len(gb) > 0 and np.sum(gc["delta"]) > 0
    rep = _check(cascade, case, gc, gb, gst)
    assert rep["frames_boxes_checked"] == 2 and rep["exempt_T2"] == 0
    assert rep["boxes"] == len(gb)


@pytest.mark.parametrize("defect", ["box_x", "neighbors", "drop_accepted", "flip_delta",
                                    "count", "score"])
def test_defects_are_caught(cascade, case, defect):
    gc, gb, gst = _as_gpu(*case[4:7])
    if defect == "box_x":
        gb["x"][0] += 1
    elif defect == "neighbors":
        gb["neighbors"][0] += 1
    elif defect == "drop_accepted":
        k = int(np.nonzero(gc["delta"] == 1)[0][0])
        gc = np.delete(gc, k)
    elif defect == "flip_delta":
        k = int(np.nonzero(gc["delta"] == 1)[0][0])
        gc["delta"][k] = 0
    elif defect == "count":
        gst["stage2"] += 1
    elif defect == "score":
        gb["score"][0] += 1e-3
    with pytest.raises(AssertionError):
        _check(cascade, case, gc, gb, gst)


def test_gap_threshold_margin():
    rng = np.random.default_rng(0)
    v = rng.normal(0, 0.2, 20000)
    t, m = parity.gap_threshold(v, 500)
    assert m > parity.TOL
    assert np.min(np.abs(v - t)) >= m - 1e-12
    assert 300 < np.sum(v > t) < 700


def test_c1_exact_thresholds_leave_work(cascade):
    """smoke()'s thresholds: survivors, stage-2/3 passes and boxes all non-empty."""
    c = configs.C1
    fr = c.make_frames()
    T1, T2, m = parity.exact_thresholds(cascade, fr, c.min_face, c.scale_step, 0.98, Tnn=c.Tnn)
    assert all(x > parity.TOL for x in m)
    _, ob, st = oracle.detect(cascade, fr, c.min_face, c.scale_step, T1, T2, c.Tnn, c.rule)
    assert st["stage1"] > 100 and st["stage2"] > 10 and st["stage3"] > 10 and len(ob) > 0

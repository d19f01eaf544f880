"""GPU NMS (nms.cu, step 4 of Fig. 3 -- P:101 "aggregates the found regions"; reading O9)
through the C ABI test hook ccnn_debug_group on hand-built raw-box sets, compared bit for
bit (boxes, neighbours, float scores and output order) with the oracle's grouping
(oracle/ccnn_oracle.c or_group: all-pairs IoU test, union-find, integer means).

The sets target what the device algorithm does differently from the oracle: x-sorted
pruning of the pair tests, the concurrent lock-free union-find (long chains, dense clutter),
shared-memory atomics for the sums / max score, the rank sort (ties), the per-frame
capacity (4096) and the last-CTA compaction of many frames.
"""
import numpy as np
import pytest

import oracle
from synth import arch, weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def det():
    from paper_1508_01292_b200 import Detector
    d = Detector(arch.NETS, weights.make_cascade_weights(), 0.5, (0.5, 0.5), 2, 0,
                 max_w=640, max_h=480, max_batch=32)
    yield d
    d.close()


def raw_boxes(rows):
    """rows: (frame, x, y, w, h, score) -> ccnn BOX_DTYPE array."""
    from paper_1508_01292_b200 import BOX_DTYPE
    a = np.zeros(len(rows), BOX_DTYPE)
    for k, r in enumerate(rows):
        a[k] = (r[0], r[1], r[2], r[3], r[4], np.float32(r[5]), 0)
    return a


def oracle_groups(raw, n_frames, min_cluster=1):
    out = []
    for f in range(n_frames):
        sel = raw[raw["frame"] == f]
        for g in oracle.group([(int(b["x"]), int(b["y"]), int(b["w"]), int(b["h"]),
                                float(b["score"])) for b in sel], min_cluster):
            out.append((f, g[0], g[1], g[2], g[3], np.float32(g[4]), g[5]))
    return out


def assert_same(got, ref):
    got = [(int(b["frame"]), int(b["x"]), int(b["y"]), int(b["w"]), int(b["h"]),
            np.float32(b["score"]), int(b["neighbors"])) for b in got]
    assert len(got) == len(ref), (len(got), len(ref))
    for k, (g, r) in enumerate(zip(got, ref)):
        assert g == r, (k, g, r)


def test_iou_exactly_0_3_is_an_edge(det):
    """w = 13, dx = 7: inter = 6h, union = 20h -> 10*inter == 3*union (IoU = 0.3 exactly:
    an edge); dx = 8: IoU = 5/21 < 0.3 (no edge)."""
    raw = raw_boxes([(0, 100, 50, 13, 20, 0.5), (0, 107, 50, 13, 20, 0.25),
                     (1, 100, 50, 13, 20, 0.5), (1, 108, 50, 13, 20, 0.25)])
    got = det.group(raw, 2)
    ref = oracle_groups(raw, 2)
    assert [r[6] for r in ref] == [2, 1, 1]
    assert_same(got, ref)


def test_long_chains(det):
    """Each box overlaps only its neighbours at IoU exactly 0.3: chains of 300 / 1000 boxes
    (in shuffled arrival order) must become one group each; a second chain in y."""
    rng = np.random.default_rng(3)
    rows = [(0, 7 * i, 40, 13, 20, float(rng.random())) for i in range(300)]
    rows += [(0, 30, 200 + 7 * i, 20, 13, float(rng.random())) for i in range(200)]
    rows += [(1, 7 * i, 10, 13, 20, float(rng.random())) for i in range(1000)]
    rng.shuffle(rows)
    raw = raw_boxes(rows)
    got = det.group(raw, 2)
    ref = oracle_groups(raw, 2)
    assert sorted(r[6] for r in ref) == [200, 300, 1000]
    assert_same(got, ref)


def test_duplicates_and_score_ties(det):
    """identical boxes (one group each), equal scores across groups (order by y, x, w, h)."""
    rows = [(0, 10, 10, 30, 34, 0.75)] * 12 + [(0, 200, 10, 30, 34, 0.75)] * 3 + \
        [(0, 100, 5, 30, 34, 0.75), (0, 100, 300, 30, 34, 0.75), (0, 100, 300, 31, 34, 0.75)]
    raw = raw_boxes(rows)
    assert_same(det.group(raw, 1), oracle_groups(raw, 1))


def _clutter(rng, n_frames, per_frame, extent=3840, sizes=(60, 240)):
    """clusters of jittered boxes (a detection's neighbourhood: position +-w/8, size +-10%),
    cluster centres uniform over a 16:9 frame, about 8 boxes per cluster."""
    rows = []
    for f in range(n_frames):
        n = per_frame if np.isscalar(per_frame) else per_frame[f]
        nc = max(1, n // 8)
        cx = rng.integers(0, extent, nc)
        cy = rng.integers(0, extent * 9 // 16, nc)
        cw = rng.integers(*sizes, nc)
        for _ in range(n):
            c = rng.integers(nc)
            w = max(1, int(cw[c] * rng.uniform(0.9, 1.1)))
            h = int(w * 31 / 27 + 0.5)
            x = max(0, int(cx[c] + rng.normal(0, cw[c] / 8)))
            y = max(0, int(cy[c] + rng.normal(0, cw[c] / 8)))
            rows.append((f, x, y, w, h, float(np.float32(rng.uniform(-1.7, 1.7)))))
    return rows


@pytest.mark.parametrize("per_frame", [600, 2000, 4096])
def test_clutter_sets(det, per_frame):
    """many overlapping boxes per frame (> 512 up to the 4096 capacity), clustered like
    cluttered-scene detections; 4 frames, one of them empty."""
    rng = np.random.default_rng(per_frame)
    rows = _clutter(rng, 4, [per_frame, per_frame // 3, 0, 7])
    raw = raw_boxes(rows)
    got = det.group(raw, 4)
    ref = oracle_groups(raw, 4)
    assert len(ref) > 10
    assert_same(got, ref)
    # arrival order does not matter (integer sums; order-free components)
    perm = raw[rng.permutation(len(raw))]
    assert_same(det.group(perm, 4), ref)


def test_many_frames_compaction(det):
    """32 frames (last-CTA compaction), random sizes including frames without boxes."""
    rng = np.random.default_rng(9)
    per = [int(v) for v in rng.integers(0, 300, 32)]
    per[5] = per[17] = 0
    raw = raw_boxes(_clutter(rng, 32, per, extent=1920))
    assert_same(det.group(raw, 32), oracle_groups(raw, 32))


def test_capacity_and_arguments(det):
    from paper_1508_01292_b200 import ccnn
    rng = np.random.default_rng(1)
    raw = raw_boxes(_clutter(rng, 1, 4097))
    with pytest.raises(ccnn.CcnnError) as e:
        det.group(raw, 1)
    assert e.value.code == ccnn.CCNN_E_QUEUE
    for bad in [(0, -1, 0, 10, 10, 0.0), (0, 0, 0, 0, 10, 0.0), (1, 0, 0, 10, 10, 0.0),
                (0, 32760, 0, 10, 10, 0.0), (0, 0, 0, 10, 10, float("nan"))]:
        with pytest.raises(ccnn.CcnnError) as e:
            det.group(raw_boxes([bad]), 1)
        assert e.value.code == ccnn.CCNN_E_ARG
    assert len(det.group(raw_boxes([]), 1)) == 0


def test_min_cluster(det):
    from paper_1508_01292_b200 import Detector
    d3 = Detector(arch.NETS, weights.make_cascade_weights(), 0.5, (0.5, 0.5), 2, 0,
                  nms_min_cluster=3, max_w=640, max_h=480, max_batch=4)
    rng = np.random.default_rng(5)
    raw = raw_boxes(_clutter(rng, 2, 500, extent=1920))
    assert_same(d3.group(raw, 2), oracle_groups(raw, 2, min_cluster=3))
    d3.close()

"""The NEXT #3 scoring harness (paper_1508_01292_b200/evaluate.py) against the SPEC
evalharness examples, closed forms, brute force and invariants."""
import itertools
import math

import numpy as np
import pytest

from paper_1508_01292_b200 import evaluate as ev
from synth import frames as synth_frames


def test_iou_rect_examples_and_invariants():
    assert ev.iou_rect((3, 4, 10, 12), (3, 4, 10, 12)) == 1.0
    assert ev.iou_rect((0, 0, 10, 10), (20, 0, 10, 10)) == 0.0
    assert ev.iou_rect((0, 0, 10, 10), (5, 0, 10, 10)) == pytest.approx(50 / 150)
    rng = np.random.default_rng(7)
    for _ in range(300):
        a = tuple(rng.uniform(1, 50, 4))
        b = tuple(rng.uniform(1, 50, 4))
        v = ev.iou_rect(a, b)
        assert 0.0 <= v <= 1.0 and v == pytest.approx(ev.iou_rect(b, a))
        # brute force on a fine grid of the joint box
        if v > 0:
            xs = np.linspace(min(a[0], b[0]), max(a[0] + a[2], b[0] + b[2]), 400)
            ys = np.linspace(min(a[1], b[1]), max(a[1] + a[3], b[1] + b[3]), 400)
            X, Y = np.meshgrid(xs, ys)
            ia = (X >= a[0]) & (X < a[0] + a[2]) & (Y >= a[1]) & (Y < a[1] + a[3])
            ib = (X >= b[0]) & (X < b[0] + b[2]) & (Y >= b[1]) & (Y < b[1] + b[3])
            assert abs(np.count_nonzero(ia & ib) / np.count_nonzero(ia | ib) - v) < 0.03
    m = ev.iou_matrix([(0, 0, 10, 10), (5, 5, 4, 4)], [(5, 0, 10, 10), (0, 0, 10, 10), (100, 100, 1, 1)])
    for i, a in enumerate([(0, 0, 10, 10), (5, 5, 4, 4)]):
        for j, b in enumerate([(5, 0, 10, 10), (0, 0, 10, 10), (100, 100, 1, 1)]):
            assert m[i, j] == pytest.approx(ev.iou_rect(a, b))


def test_iou_ellipse_rect_examples():
    # ellipse well inside a huge rectangle: area(e) / area(r), within 2% of pi a b / area(r)
    r = (0, 0, 200, 200)
    v = ev.iou_ellipse_rect((30, 20, 0.0, 100, 100), r)
    assert v == pytest.approx(math.pi * 30 * 20 / 200 ** 2, rel=0.02)
    # disjoint bounding boxes -> 0
    assert ev.iou_ellipse_rect((10, 5, 0.3, 0, 0), (100, 100, 10, 10)) == 0.0
    # circle of radius 10 vs its bounding square: pi / 4 +- 0.02; rotation-invariant
    for th in (0.0, 0.7, 2.0):
        assert ev.iou_ellipse_rect((10, 10, th, 50, 50), (40, 40, 20, 20)) == pytest.approx(math.pi / 4, abs=0.02)
    # finer grid converges to the same value
    a = ev.iou_ellipse_rect((25, 15, 0.5, 60, 50), (40, 35, 40, 30))
    b = ev.iou_ellipse_rect((25, 15, 0.5, 60, 50), (40, 35, 40, 30), step=0.5)
    assert abs(a - b) < 0.01


def _brute_greedy(iou, thr):
    """Independent form of E2: repeatedly take the largest remaining IoU (first in row-major
    order on ties) and delete its row and column."""
    m = np.where(iou > thr, iou, -1.0).astype(np.float64)
    pairs = []
    while m.size and m.max() > thr:
        a, d = np.unravel_index(int(np.argmax(m)), m.shape)
        pairs.append((int(a), int(d)))
        m[a, :] = -1
        m[:, d] = -1
    return sorted(pairs)


def test_match_discrete_examples_and_brute_force():
    ann = [(0, 0, 10, 10), (30, 30, 12, 14), (60, 0, 8, 8)]
    pairs, fn, fp = ev.match_discrete(ann, ann)
    assert len(pairs) == 3 and fn == [] and fp == []
    # sole detection with IoU 0.4 -> 1 FP and 1 FN
    det = (0, 0, 10, 10)
    ann1 = (0, 0, 10, 4)                                                  # IoU = 40 / 100
    assert ev.iou_rect(ann1, det) == pytest.approx(0.4)
    pairs, fn, fp = ev.match_discrete([ann1], [det])
    assert pairs == [] and fn == [0] and fp == [0]
    # IoU exactly 0.5 does not "exceed" 0.5 (E1)
    pairs, _, _ = ev.match_discrete([(0, 0, 10, 10)], [(0, 0, 10, 5)])
    assert pairs == []
    # crafted 4x4 IoU matrix where greedy differs from the maximum-cardinality matching
    iou = np.array([[0.9, 0.8, 0.0, 0.0], [0.85, 0.0, 0.0, 0.0],
                    [0.0, 0.0, 0.6, 0.7], [0.0, 0.0, 0.65, 0.0]])
    pairs, fn, fp = ev.match_greedy(iou)
    assert sorted((a, d) for a, d, _ in pairs) == [(0, 0), (2, 3), (3, 2)] == _brute_greedy(iou, 0.5)
    assert fn == [1] and fp == [1]
    rng = np.random.default_rng(3)
    for _ in range(200):
        m = np.round(rng.uniform(0, 1, (rng.integers(0, 6), rng.integers(0, 6))), 2)
        pairs, fn, fp = ev.match_greedy(m)
        got = sorted((a, d) for a, d, _ in pairs)
        assert got == _brute_greedy(m, 0.5)
        # one-to-one, and the unmatched lists complete the index sets
        assert len({a for a, _ in got}) == len(got) == len({d for _, d in got})
        assert sorted([a for a, _ in got] + fn) == list(range(m.shape[0]))
        assert sorted([d for _, d in got] + fp) == list(range(m.shape[1]))


def test_score_fddb_examples_and_monotone():
    ann = [[(0, 0, 10, 10)], [(20, 20, 10, 10), (50, 50, 10, 10)]]
    # perfect detector: TPR 1 at FP 0 below the minimum score
    imgs = [(a, a, [0.9] * len(a)) for a in ann]
    rows = ev.score_fddb(imgs, [0.0, 0.5, 0.89])
    assert all(r["tpr"] == 1.0 and r["fp"] == 0 and r["continuous"] == 1.0 for r in rows)
    # empty detections: TPR 0, FP 0, continuous 0
    rows = ev.score_fddb([(a, np.zeros((0, 4)), []) for a in ann], [0.0])
    assert rows[0] == dict(threshold=0.0, tpr=0.0, fp=0, continuous=0.0)
    # 5-image hand-enumerated fixture
    imgs = [
        ([(0, 0, 10, 10)], [(0, 0, 10, 10)], [0.9]),                      # TP iou 1 @0.9
        ([(0, 0, 10, 10)], [(0, 0, 10, 8), (50, 50, 5, 5)], [0.8, 0.3]),   # TP iou .8 @.8, FP @.3
        ([(0, 0, 10, 10)], [(0, 0, 10, 4)], [0.7]),                       # iou .4: FP @.7, FN
        ([], [(5, 5, 5, 5)], [0.6]),                                      # FP @.6
        ([(0, 0, 10, 10), (20, 0, 10, 10)], [(20, 0, 10, 10)], [0.2]),    # TP iou 1 @.2, FN
    ]
    rows = {r["threshold"]: r for r in ev.score_fddb(imgs, [0.0, 0.25, 0.65, 0.75, 0.85, 0.95])}
    table = {0.0: (3, 3, 2.8), 0.25: (2, 3, 1.8), 0.65: (2, 1, 1.8), 0.75: (2, 0, 1.8),
             0.85: (1, 0, 1.0), 0.95: (0, 0, 0.0)}
    for t, (tp, fp, cont) in table.items():
        assert rows[t]["tpr"] == pytest.approx(tp / 5) and rows[t]["fp"] == fp
        assert rows[t]["continuous"] == pytest.approx(cont / 5)
    fps = [rows[t]["fp"] for t in sorted(rows)]
    assert fps == sorted(fps, reverse=True)                               # monotone ROC


def test_multiscale_examples_and_monotone():
    a = (100, 100, 40, 46)
    assert ev.match_multiscale(a, a)
    cx, cy = 120, 123
    d = (cx - 1.15 * 20, cy - 1.15 * 23, 1.15 * 40, 1.15 * 46)
    assert ev.match_multiscale(a, d)
    best = max(ev.iou_rect(v, d) for v in ev.scaled_variants(a))
    assert best > 0.95                                                    # a factor near 1.15 exists
    big = (cx - 3 * 20, cy - 3 * 23, 120, 138)                             # 3x -> no match
    assert not ev.match_multiscale(a, big)
    assert max(ev.iou_rect(v, big) for v in ev.scaled_variants(a, np.linspace(0.9, 1.2, 1000))) < 0.5
    assert len(ev.AFW_FACTORS) == 44 and ev.AFW_FACTORS[0] == 0.9
    assert ev.AFW_FACTORS[-1] == pytest.approx(1.2)
    # adding variants never turns a match into a non-match
    rng = np.random.default_rng(11)
    for _ in range(200):
        dd = tuple(rng.uniform(60, 160, 2)) + tuple(rng.uniform(20, 70, 2))
        few = ev.match_multiscale(a, dd, factors=ev.AFW_FACTORS[::7])
        assert (not few) or ev.match_multiscale(a, dd)


def test_prf1_examples():
    assert ev.prf1(4, 0, 0) == (1.0, 1.0, 1.0)
    assert ev.prf1(0, 0, 3) == (0.0, 0.0, 0.0)
    assert ev.prf1(3, 1, 1) == pytest.approx((0.75, 0.75, 0.75))
    r = ev.score_afw([([(0, 0, 10, 10), (50, 50, 10, 10)], [(0, 0, 10, 10), (30, 30, 5, 5)])])
    assert (r["tp"], r["fp"], r["fn"]) == (1, 1, 1) and r["f1"] == pytest.approx(0.5)


def test_make_still_gt_matches_make_still():
    img, gt = synth_frames.make_still_gt(333, 257, 991, 20)
    assert np.array_equal(img, synth_frames.make_still(333, 257, 991, 20))
    assert len(gt) >= 1
    for x, y, w, h in gt:
        assert 0 <= x and x + w <= 333 and 0 <= y and y + h <= 257 and h == (w * 23) // 20

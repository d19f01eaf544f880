"""Pins for the oracle's grouping / NMS (SPEC group_detections S:329-337).

Checked against the SPEC worked examples, an exact-rational IoU, and a brute-force
BFS connected-components grouping on tiny random sets, plus permutation invariance.
"""
from fractions import Fraction

import numpy as np

import oracle

RNG = np.random.default_rng(5)


def _iou(a, b):
    ix = min(a[0] + a[2], b[0] + b[2]) - max(a[0], b[0])
    iy = min(a[1] + a[3], b[1] + b[3]) - max(a[1], b[1])
    if ix <= 0 or iy <= 0:
        return Fraction(0)
    inter = ix * iy
    return Fraction(inter, a[2] * a[3] + b[2] * b[3] - inter)


def _brute_group(boxes, min_cluster):
    n = len(boxes)
    seen = [False] * n
    out = []
    for s in range(n):
        if seen[s]:
            continue
        comp, stack = [], [s]
        seen[s] = True
        while stack:
            a = stack.pop()
            comp.append(a)
            for b in range(n):
                if not seen[b] and _iou(boxes[a], boxes[b]) >= Fraction(3, 10):
                    seen[b] = True
                    stack.append(b)
        if len(comp) < min_cluster:
            continue
        k = len(comp)
        mean = [int(Fraction(sum(boxes[c][q] for c in comp), k) + Fraction(1, 2)) for q in range(4)]
        out.append((*mean, max(boxes[c][4] for c in comp), k))
    out.sort(key=lambda b: (-b[4], b[1], b[0], b[2], b[3]))
    return out


def test_iou_example(golden):
    ex = golden["iou_example"]
    assert _iou(ex["a"], ex["b"]) == Fraction(*ex["iou"])
    assert oracle.iou_edge(ex["a"], ex["b"])                      # 1/3 >= 0.3
    # exactly 0.3 is an edge, just below is not: a=(0,0,10,10), b=(x,0,10,10)
    # IoU = (10-x)*10 / (200 - (10-x)*10); = 0.3 at (10-x)*10 = 600/13 (not integral) ->
    # use heights: a=(0,0,13,10), b=(0,0,13,h) ...; direct search for an exact 3/10 case
    found = False
    for w1 in range(1, 40):
        for w2 in range(1, 40):
            a, b = (0, 0, w1, 10), (0, 0, w2, 10)
            if _iou(a, b) == Fraction(3, 10):
                assert oracle.iou_edge(a, b)
                found = True
    assert found


def test_spec_examples(golden):
    assert oracle.group([], 1) == []
    ex = golden["grouping_examples"]["three_plus_isolated"]
    boxes = [tuple(b) + (0.5 + 0.1 * k,) for k, b in enumerate(ex["boxes"])]
    out = oracle.group(boxes, ex["min_cluster"])
    assert len(out) == ex["n_out"] and out[0][5] == ex["neighbors"]
    three = np.array(ex["boxes"][:3])
    assert out[0][:4] == tuple(int(np.floor(m + 0.5)) for m in three.mean(axis=0))
    ex = golden["grouping_examples"]["disjoint"]
    boxes = [tuple(b) + (0.1 * k,) for k, b in enumerate(ex["boxes"])]
    out = oracle.group(boxes, 1)
    assert sorted(o[:4] for o in out) == sorted(tuple(b) for b in ex["boxes"])
    assert all(o[5] == 1 for o in out)


def test_group_vs_brute_force():
    for trial in range(150):
        n = int(RNG.integers(0, 12))
        boxes = []
        for _ in range(n):
            w = int(RNG.integers(5, 30))
            boxes.append((int(RNG.integers(0, 60)), int(RNG.integers(0, 60)), w,
                          w + int(RNG.integers(0, 6)), float(RNG.normal())))
        mc = int(RNG.integers(1, 4))
        got = oracle.group(boxes, mc)
        ref = _brute_group(boxes, mc)
        assert got == ref
        perm = RNG.permutation(n)
        assert oracle.group([boxes[k] for k in perm], mc) == got     # order-free

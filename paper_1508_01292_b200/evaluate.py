"""Detection-quality scoring on synthetic ground truth.

Host-side protocol code that scores the boxes the detector returned -- it is not a step of
the detection path (every step of that runs in libccnn.so) and it never produces boxes.
It follows the paper's two benchmark protocols, applied to planted synthetic faces
(`synth.frames.make_still_gt`) because the real FDDB / AFW sets are out of scope:

* FDDB (§4.1): a detection is positive if the IoU with an annotation *exceeds* 0.5;
  one detection per annotation; the discrete score is the ROC of detected fraction vs false
  alarms over a sweep of the decision threshold, the continuous score the average IoU.
  Annotations may be rectangles or FDDB-style ellipses (rasterised IoU).
* AFW (§4.2): precision / recall / F1 with the IoU-0.5 test against the
  annotation and 44 centre-preserving rescaled copies of it (factors 0.9 .. 1.2), averaged
  over minNeighbors = {1, 2, 3} (== T_nn).

Readings (E1-E4): E1 "exceeds 0.5" is strict (IoU > 0.5) in both protocols;
E2 one-to-one matching is greedy by descending IoU (ties: lower annotation index, then lower
detection index); E3 the 44 factors are 0.9 + i * 0.3 / 43, i = 0..43 (the paper gives
only the endpoints and the count); E4 ellipse IoU is rasterised on the unit-pixel grid of
the joint bounding box (pixel centres), continuous score = sum of matched IoU / #annotations,
precision with no detections = 0, F1 with P + R = 0 = 0.
"""
import math

import numpy as np

IOU_THRESHOLD = 0.5
AFW_FACTORS = tuple(0.9 + i * 0.3 / 43 for i in range(44))


def iou_rect(a, b) -> float:
    """IoU of two rectangles (x, y, w, h) with positive extents (continuous coordinates)."""
    ax, ay, aw, ah = (float(v) for v in a)
    bx, by, bw, bh = (float(v) for v in b)
    iw = min(ax + aw, bx + bw) - max(ax, bx)
    ih = min(ay + ah, by + bh) - max(ay, by)
    inter = max(iw, 0.0) * max(ih, 0.0)
    union = aw * ah + bw * bh - inter
    return inter / union if union > 0 else 0.0


def iou_matrix(annots, dets) -> np.ndarray:
    """(len(annots), len(dets)) rectangle IoUs."""
    A = np.asarray(annots, np.float64).reshape(-1, 4)
    D = np.asarray(dets, np.float64).reshape(-1, 4)
    if len(A) == 0 or len(D) == 0:
        return np.zeros((len(A), len(D)))
    ix = np.minimum(A[:, None, 0] + A[:, None, 2], D[None, :, 0] + D[None, :, 2]) - \
        np.maximum(A[:, None, 0], D[None, :, 0])
    iy = np.minimum(A[:, None, 1] + A[:, None, 3], D[None, :, 1] + D[None, :, 3]) - \
        np.maximum(A[:, None, 1], D[None, :, 1])
    inter = np.clip(ix, 0, None) * np.clip(iy, 0, None)
    union = (A[:, 2] * A[:, 3])[:, None] + (D[:, 2] * D[:, 3])[None, :] - inter
    return np.where(union > 0, inter / np.where(union > 0, union, 1.0), 0.0)


def iou_ellipse_rect(e, r, step: float = 1.0) -> float:
    """IoU of an ellipse (major radius, minor radius, angle [rad], cx, cy) -- FDDB's
    annotation format, major axis along the angle -- and a rectangle (x, y, w, h), by
    rasterisation at the centres of a `step`-pixel grid over the joint bounding box (E4)."""
    ra, rb, th, cx, cy = (float(v) for v in e)
    x, y, w, h = (float(v) for v in r)
    c, s = math.cos(th), math.sin(th)
    ex = math.sqrt((ra * c) ** 2 + (rb * s) ** 2)       # ellipse bounding half-extents
    ey = math.sqrt((ra * s) ** 2 + (rb * c) ** 2)
    x0, x1 = min(cx - ex, x), max(cx + ex, x + w)
    y0, y1 = min(cy - ey, y), max(cy + ey, y + h)
    xs = x0 + (np.arange(max(1, int(math.ceil((x1 - x0) / step)))) + 0.5) * step
    ys = y0 + (np.arange(max(1, int(math.ceil((y1 - y0) / step)))) + 0.5) * step
    X, Y = np.meshgrid(xs, ys)
    u = (X - cx) * c + (Y - cy) * s
    v = -(X - cx) * s + (Y - cy) * c
    in_e = (u / ra) ** 2 + (v / rb) ** 2 <= 1.0
    in_r = (X >= x) & (X < x + w) & (Y >= y) & (Y < y + h)
    union = np.count_nonzero(in_e | in_r)
    return np.count_nonzero(in_e & in_r) / union if union else 0.0


def match_greedy(iou: np.ndarray, threshold: float = IOU_THRESHOLD):
    """One-to-one greedy matching on an (annotations x detections) IoU matrix (E2): pairs
    taken by descending IoU while IoU > threshold.  Returns (pairs [(a, d, iou)], unmatched
    annotation indices, unmatched detection indices)."""
    na, nd = iou.shape
    cand = [(-iou[a, d], a, d) for a in range(na) for d in range(nd) if iou[a, d] > threshold]
    cand.sort()
    ua, ud, pairs = set(range(na)), set(range(nd)), []
    for negv, a, d in cand:
        if a in ua and d in ud:
            pairs.append((a, d, -negv))
            ua.discard(a)
            ud.discard(d)
    return pairs, sorted(ua), sorted(ud)


def match_discrete(annots, dets, threshold: float = IOU_THRESHOLD):
    """FDDB discrete matching of rectangles: see match_greedy."""
    return match_greedy(iou_matrix(annots, dets), threshold)


def score_fddb(images, thresholds):
    """FDDB discrete ROC + continuous score.

    images: iterable of (annotations [rects], detections [rects], scores [floats]).
    For every threshold t (detections with score >= t kept): detected fraction (TPR) and
    total false alarms; continuous = sum of matched IoU / #annotations.
    Returns a list of dicts {threshold, tpr, fp, continuous}."""
    images = [(np.asarray(a, np.float64).reshape(-1, 4), np.asarray(d, np.float64).reshape(-1, 4),
               np.asarray(s, np.float64).reshape(-1)) for a, d, s in images]
    n_ann = sum(len(a) for a, _, _ in images)
    rows = []
    for t in thresholds:
        tp = fp = 0
        cont = 0.0
        for a, d, s in images:
            keep = s >= t
            pairs, _, ud = match_discrete(a, d[keep])
            tp += len(pairs)
            fp += len(ud)
            cont += sum(p[2] for p in pairs)
        rows.append(dict(threshold=float(t), tpr=tp / n_ann if n_ann else 0.0, fp=fp,
                         continuous=cont / n_ann if n_ann else 0.0))
    return rows


def scaled_variants(annot, factors=AFW_FACTORS):
    """Centre-preserving rescaled copies of a rectangle annotation (E3)."""
    x, y, w, h = (float(v) for v in annot)
    cx, cy = x + w / 2, y + h / 2
    return [(cx - f * w / 2, cy - f * h / 2, f * w, f * h) for f in factors]


def multiscale_iou(annot, det, factors=AFW_FACTORS) -> float:
    """Best IoU of the detection against the annotation and its rescaled copies."""
    return max([iou_rect(annot, det)] + [iou_rect(v, det) for v in scaled_variants(annot, factors)])


def match_multiscale(annot, det, threshold: float = IOU_THRESHOLD, factors=AFW_FACTORS) -> bool:
    """AFW match test: IoU > threshold against any variant (or the original)."""
    return multiscale_iou(annot, det, factors) > threshold


def prf1(tp: int, fp: int, fn: int):
    """(precision, recall, F1) with 0 for the undefined cases (E4)."""
    p = tp / (tp + fp) if tp + fp else 0.0
    r = tp / (tp + fn) if tp + fn else 0.0
    f = 2 * p * r / (p + r) if p + r else 0.0
    return p, r, f


def score_afw(images, factors=AFW_FACTORS):
    """AFW precision / recall / F1 over images [(annotations, detections)],
    one-to-one greedy matching on the multi-scale IoU.  Returns dict(tp, fp, fn, precision,
    recall, f1)."""
    tp = fp = fn = 0
    for annots, dets in images:
        A = np.asarray(annots, np.float64).reshape(-1, 4)
        D = np.asarray(dets, np.float64).reshape(-1, 4)
        m = np.array([[multiscale_iou(a, d, factors) for d in D] for a in A]).reshape(len(A), len(D))
        pairs, ua, ud = match_greedy(m)
        tp += len(pairs)
        fp += len(ud)
        fn += len(ua)
    p, r, f = prf1(tp, fp, fn)
    return dict(tp=tp, fp=fp, fn=fn, precision=p, recall=r, f1=f)


def boxes_by_frame(boxes, n_frames):
    """Split a ccnn box array (BOX_DTYPE) into per-frame (rects, scores, neighbors)."""
    out = []
    for f in range(n_frames):
        b = boxes[boxes["frame"] == f]
        out.append((np.stack([b["x"], b["y"], b["w"], b["h"]], 1).astype(np.float64)
                    if len(b) else np.zeros((0, 4)), b["score"].astype(np.float64),
                    b["neighbors"].astype(np.int64)))
    return out

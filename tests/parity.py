"""Parity helpers: compare the CUDA path (through the C ABI) with the oracle.

Bar (BASELINE.json north_star):
* pyramid levels and every integer / geometry quantity: bit-exact;
* per-window stage-1 scores and all CNN2/CNN3 responses: |gpu - oracle| <= 1e-4;
* survivor sets, K2/K3, delta, raw boxes, final boxes and the Table-1 counts: exact, except
  the decisions of windows whose oracle score lies within 1e-4 of T1 and of candidates with
  a response within 1e-4 of T2 ("exempt"): for those -- and only those -- either decision is
  correct.

Every frame's final boxes and every run's Table-1 counts are compared (no frame is dropped):
the reference is the oracle's grouping (or_group, P:101 reading O9) of the oracle's accepted
raw boxes, where an exempt decision is taken as the GPU took it.  Without exemptions that
reference IS the oracle's own detection (asserted).  Tests place their thresholds with
`exact_thresholds` (largest-gap placement on the test frames themselves, margin > 1e-4), so
they normally have no exemption at all; the reports count them.

Independently, `check_nms` runs the oracle's grouping on the GPU's own accepted raw boxes
and GPU scores: the GPU's boxes must equal it bit for bit, order included (no tolerance:
the NMS input is identical on both sides).
"""
import os

import numpy as np

import oracle

TOL = 1e-4


def key(c):
    return (int(c["frame"]), int(c["level"]), int(c["iy"]), int(c["ix"]))


class Report(dict):
    pass


def _pmap(fn, items):
    """map over a thread pool (the oracle's C calls release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    items = list(items)
    with ThreadPoolExecutor(max(1, min(len(items), os.cpu_count() or 1))) as pool:
        return list(pool.map(fn, items))


def oracle_maps(cascade, frames, min_face, scale_step):
    """{(frame, level): dense oracle stage-1 map} and the oracle level table."""
    lv = oracle.level_table(frames.shape[2], frames.shape[1], min_face, scale_step)
    jobs = [(f, l) for f in range(frames.shape[0]) for l in range(len(lv))]
    res = _pmap(lambda fl: oracle.stage1_dense(cascade.nets[0], oracle.resample(
        frames[fl[0]], *lv[fl[1]])), jobs)
    return lv, dict(zip(jobs, res))


# ---------------------------------------------------------------------------------------
# threshold placement with a margin (test inputs only; calibration: oracle/calibrate.py)
# ---------------------------------------------------------------------------------------
def gap_threshold(values, n_above, min_margin=1.5 * TOL, window=0.25):
    """float32 threshold with about n_above of `values` strictly above it, at the midpoint of
    the largest gap between consecutive sorted values within +-window of that rank (widened
    until the margin to the nearest value exceeds min_margin).  Returns (T, margin)."""
    v = np.unique(np.asarray(values, np.float64))[::-1]          # descending, distinct
    if len(v) < 2:
        raise ValueError("need at least 2 distinct values")
    n_above = min(max(1, int(round(n_above))), len(v) - 1)
    best = None
    for win in (window, 0.5, 0.75, 1.0):
        lo = max(1, int(np.floor((1 - win) * n_above)))
        hi = min(len(v) - 1, max(lo, int(np.ceil((1 + win) * n_above))))
        gaps = v[lo - 1:hi] - v[lo:hi + 1]
        k = lo + int(np.argmax(gaps))
        t = float(np.float32(0.5 * (v[k - 1] + v[k])))
        margin = float(min(abs(v[k - 1] - t), abs(v[k] - t)))
        if best is None or margin > best[1]:
            best = (t, margin)
        if margin > min_margin:
            break
    return best


def exact_thresholds(cascade, frames, min_face, scale_step, q1, rule=0, Tnn=2, p2=0.5, p3=0.6):
    """(T1, (T2a, T2b), margins) placed on the test frames themselves so that no window lies
    within 1e-4 of T1 and no CNN2 / CNN3 response of a survivor within 1e-4 of T2a / T2b.
    q1: stage-1 quantile (fraction of windows rejected); p2 ~ P(K2 > 0); p3 ~ P(delta = 1)."""
    frames = [np.ascontiguousarray(f, np.uint8) for f in frames]
    vals = []
    for fr in frames:
        _, maps = oracle_maps(cascade, fr[None], min_face, scale_step)
        vals += [m.ravel() for m in maps.values()]
    vals = np.concatenate(vals)
    T1, m1 = gap_threshold(vals, (1.0 - q1) * vals.size)
    # every survivor's responses: CNN3 runs for all of them when T2a is below the range
    cands = np.concatenate([oracle.detect(cascade, fr[None], min_face, scale_step, T1,
                                          (-10.0, -10.0), Tnn, 0)[0] for fr in frames])
    if len(cands) == 0:
        return T1, (0.5, 0.5), (m1, None, None)
    r2 = cands["r2"]
    # T2a near the value that gives K2 > 0 for a fraction p2 of the candidates
    target = np.quantile(r2.max(axis=1), 1.0 - p2)
    T2a, m2 = gap_threshold(r2.ravel(), np.sum(r2.ravel() > target))
    K2 = np.sum(r2.astype(np.float32) > np.float32(T2a), axis=1)
    runs3 = (K2 > 0) if rule == 0 else (K2 < Tnn)
    if not np.any(runs3):
        return T1, (T2a, 0.5), (m1, m2, None)
    r3 = cands["r3"][runs3]
    r3s = -np.sort(-r3, axis=1)
    target3 = np.quantile(r3s[:, min(Tnn, 50) - 1], 1.0 - p3)
    T2b, m3 = gap_threshold(r3.ravel(), np.sum(r3.ravel() > target3))
    return T1, (T2a, T2b), (m1, m2, m3)


# ---------------------------------------------------------------------------------------
# comparisons
# ---------------------------------------------------------------------------------------
def _box_tuples(boxes):
    return sorted((int(b["x"]), int(b["y"]), int(b["w"]), int(b["h"]), int(b["neighbors"]),
                   float(b["score"])) for b in boxes)


def check_nms(gc, gboxes, n_frames):
    """The GPU's NMS output equals the oracle's grouping (or_group) of the GPU's own accepted
    raw boxes with the GPU's scores, bit for bit and in the same order, on every frame.
    Returns (frames checked, raw boxes grouped)."""
    acc = gc[gc["delta"] == 1]
    n_raw = 0
    for f in range(n_frames):
        a = acc[acc["frame"] == f]
        n_raw += len(a)
        ref = oracle.group([(int(x["bx"]), int(x["by"]), int(x["bw"]), int(x["bh"]),
                             float(x["score"])) for x in a])
        got = gboxes[gboxes["frame"] == f]
        assert len(got) == len(ref), f"frame {f}: {len(got)} groups vs or_group {len(ref)}"
        for g, r in zip(got, ref):
            assert (int(g["x"]), int(g["y"]), int(g["w"]), int(g["h"]), int(g["neighbors"])) == \
                tuple(r[:4]) + (r[5],), f"frame {f}: {g} vs {r}"
            assert np.float32(g["score"]) == np.float32(r[4]), f"frame {f}: score {g} vs {r}"
    return n_frames, n_raw


def _near(vals, T):
    return bool(np.any(np.abs(np.asarray(vals, np.float64) - T) <= TOL))


def check_selective_and_boxes(gc, gboxes, gstats, ocands, oboxes, ostats, exempt1, frames,
                              lvs, cascade, T1, T2, Tnn, rule, frame_ids=None, rep=None):
    """Survivor sets, per-candidate selective outcome, final boxes of EVERY frame in
    `frame_ids` (default: all) and -- when gstats is given -- the Table-1 counts.

    gc / gboxes: the GPU's candidates / boxes restricted to the checked frames; ocands /
    oboxes / ostats: oracle.detect over the same frames (frame ids matching); exempt1: the
    (frame, level, iy, ix) windows whose oracle score lies within 1e-4 of T1."""
    rep = Report() if rep is None else rep
    frame_ids = list(range(len(frames))) if frame_ids is None else list(frame_ids)
    params = oracle.make_params(T1, T2, Tnn, rule)
    gmap = {key(c): c for c in gc}
    omap = {key(c): c for c in ocands}
    assert set(gmap) - exempt1 == set(omap) - exempt1, \
        f"survivors differ: gpu-only {sorted(set(gmap) - set(omap) - exempt1)[:5]} " \
        f"oracle-only {sorted(set(omap) - set(gmap) - exempt1)[:5]}"
    # reference selective outcome for every GPU survivor (the reference survivor set is the
    # oracle's, with exempt windows decided as the GPU decided them: exactly the GPU's set)
    max_r, n_ex2 = 0.0, 0
    ref_acc = {f: [] for f in frame_ids}
    ref_counts = dict(stage1=0, stage2=0, stage3=0)
    exempt_frames = {k[0] for k in exempt1 if k in gmap or k in omap}
    for k, g in gmap.items():
        f, l, i, j = k
        if k in omap:
            o = omap[k]
            o_r2, o_r3, o = np.asarray(o["r2"]), np.asarray(o["r3"]), dict(
                K2=int(o["K2"]), K3=int(o["K3"]), delta=int(o["delta"]), cnn3_ran=int(o["cnn3_ran"]),
                score=float(o["score"]), s1=float(o["s1"]),
                box=(int(o["bx"]), int(o["by"]), int(o["bw"]), int(o["bh"])))
        else:                                   # an exempt window the GPU kept: classify it
            assert k in exempt1
            s = lvs[f][l][0]
            c = oracle.classify(cascade.nets[1], cascade.nets[2],
                                oracle.extract_patch(frames[f], s, i, j), params)
            lv = oracle.resample(frames[f], *lvs[f][l])
            o_r2, o_r3 = np.asarray(c.r2[:]), np.asarray(c.r3[:])
            o = dict(K2=c.K2, K3=c.K3, delta=c.delta, cnn3_ran=c.cnn3_ran, score=c.score,
                     s1=oracle.stage1_window(cascade.nets[0], lv, i, j),
                     box=oracle.raw_box(s, i, j))
        assert abs(float(g["s1"]) - o["s1"]) <= TOL, (k, float(g["s1"]), o["s1"])
        assert (int(g["bx"]), int(g["by"]), int(g["bw"]), int(g["bh"])) == o["box"], k
        if _has_resp(g):
            d2 = np.abs(g["r2"].astype(np.float64) - o_r2)
            max_r = max(max_r, float(d2.max()))
            assert d2.max() <= TOL, f"CNN2 responses {k}: {d2.max()}"
        near = _near(o_r2, T2[0])
        if not near:
            assert int(g["K2"]) == o["K2"] and int(g["cnn3_ran"]) == o["cnn3_ran"], (k, g["K2"], o["K2"])
            if o["cnn3_ran"]:
                if _has_resp(g):
                    d3 = np.abs(g["r3"].astype(np.float64) - o_r3)
                    max_r = max(max_r, float(d3.max()))
                    assert d3.max() <= TOL, f"CNN3 responses {k}: {d3.max()}"
                near = _near(o_r3, T2[1])
        if near:                                # either decision is correct: take the GPU's
            n_ex2 += 1
            exempt_frames.add(f)
            ref = dict(K2=int(g["K2"]), delta=int(g["delta"]), score=float(g["score"]))
        else:
            assert int(g["K3"]) == o["K3"] and int(g["delta"]) == o["delta"], (k, g, o)
            assert abs(float(g["score"]) - o["score"]) <= TOL, (k, float(g["score"]), o["score"])
            ref = dict(K2=o["K2"], delta=o["delta"], score=o["score"])
        ref_counts["stage1"] += 1
        ref_counts["stage2"] += ref["K2"] > 0
        ref_counts["stage3"] += ref["delta"] == 1
        if ref["delta"] == 1:
            ref_acc[f].append(o["box"] + (ref["score"],))
    # final boxes of every frame: oracle grouping of the reference accepted boxes
    n_boxes = 0
    for f in frame_ids:
        ref = oracle.group(ref_acc[f])
        n_boxes += len(ref)
        gb = _box_tuples(gboxes[gboxes["frame"] == f])
        rb = sorted((r[0], r[1], r[2], r[3], r[5], r[4]) for r in ref)
        assert [b[:5] for b in gb] == [b[:5] for b in rb], \
            f"frame {f}: boxes differ\n gpu {gb[:6]}\n ref {rb[:6]}"
        for a, b in zip(gb, rb):
            assert abs(a[5] - b[5]) <= TOL, (f, a, b)
        if f not in exempt_frames:              # no exemption: the reference IS the oracle's
            ob = _box_tuples(oboxes[oboxes["frame"] == f])
            assert [b[:5] for b in ob] == [b[:5] for b in rb], f"frame {f}: reference != oracle"
        ref_counts["nms"] = ref_counts.get("nms", 0) + len(ref)
    if gstats is not None:
        for k in ("stage1", "stage2", "stage3", "nms"):
            assert gstats[k] == ref_counts[k], (k, gstats[k], ref_counts[k])
        if not exempt_frames:
            for k in ("stage1", "stage2", "stage3", "nms"):
                assert gstats[k] == ostats[k], (k, gstats[k], ostats[k])
    rep["max_err_resp"] = max(rep.get("max_err_resp", 0.0), max_r)
    rep["exempt_T2"] = rep.get("exempt_T2", 0) + n_ex2
    rep["frames_boxes_checked"] = rep.get("frames_boxes_checked", 0) + len(frame_ids)
    rep["frames_with_exemptions"] = rep.get("frames_with_exemptions", 0) + len(exempt_frames)
    rep["boxes"] = rep.get("boxes", 0) + n_boxes
    rep["survivors"] = rep.get("survivors", 0) + len(gmap)
    return rep


def _has_resp(g):
    """GPU responses are only recorded with CCNN_DEBUG_STAGE1 (else the arrays are zero)."""
    return bool(np.any(g["r2"] != 0))


def _oracle_frames(cascade, frames, min_face, scale_step, T1, T2, Tnn, rule):
    """oracle.detect over a list of frames of individual sizes, frame ids = list index."""
    cands, boxes, stats = [], [], None
    for f, fr in enumerate(frames):
        c, b, st = oracle.detect(cascade, fr[None], min_face, scale_step, T1, T2, Tnn, rule)
        c["frame"] = f
        b["frame"] = f
        cands.append(c)
        boxes.append(b)
        stats = st if stats is None else {k: stats[k] + st[k] for k in stats}
    return np.concatenate(cands), np.concatenate(boxes), stats


def exempt_windows(cascade, frames, lvs, T1, frame_ids=None):
    """(frame, level, iy, ix) of every window whose dense oracle score is within 1e-4 of T1."""
    ex = set()
    jobs = [(f, l) for f in (range(len(frames)) if frame_ids is None else frame_ids)
            for l in range(len(lvs[f]))]
    maps = _pmap(lambda fl: oracle.stage1_dense(cascade.nets[0], oracle.resample(
        frames[fl[0]], *lvs[fl[0]][fl[1]])), jobs)
    for (f, l), ref in zip(jobs, maps):
        for i, j in zip(*np.nonzero(np.abs(ref - T1) <= TOL)):
            ex.add((f, l, int(i), int(j)))
    return ex


def compare_run(det, cascade, frames, min_face, scale_step, T1, T2, Tnn, rule, check_maps=True,
                check_levels=True, debug_extra=0, expect_exact=False):
    """Run the GPU detector in debug mode and the oracle on the same frames; assert parity.
    `frames`: a uint8 array (n, H, W) (ccnn_detect) or a list of 2-D frames of individual
    sizes (ccnn_detect_frames).  expect_exact: the thresholds were placed with a margin
    (exact_thresholds), so no window / response may be exempt.  Returns a Report."""
    from paper_1508_01292_b200 import ccnn
    det.set_debug(ccnn.CCNN_DEBUG_STAGE1 | ccnn.CCNN_DEBUG_LEVELS | debug_extra)
    if isinstance(frames, (list, tuple)):
        frames = [np.ascontiguousarray(f, np.uint8) for f in frames]
        gboxes = det.detect_frames(frames, min_face, scale_step)
        gstats = det.last_stats
        gc = det.candidates()
        ocands, oboxes, ostats = _oracle_frames(cascade, frames, min_face, scale_step, T1, T2,
                                                Tnn, rule)
    else:
        frames = np.ascontiguousarray(frames, np.uint8)
        if frames.ndim == 2:
            frames = frames[None]
        gboxes = det.detect(frames, min_face, scale_step)
        gstats = det.last_stats
        gc = det.candidates()
        ocands, oboxes, ostats = oracle.detect(cascade, frames, min_face, scale_step, T1, T2,
                                               Tnn, rule)
    rep = Report(n_frames=len(frames))

    # ---- level tables (per frame) and pyramid: exact ----
    lvs = [oracle.level_table(fr.shape[1], fr.shape[0], min_face, scale_step) for fr in frames]
    for f, lv in enumerate(lvs):
        glv = det.levels(f)
        assert len(glv) == len(lv), f"frame {f}: {len(glv)} levels vs {len(lv)}"
        for (gs, gw, gh), (s, w, h) in zip(glv, lv):
            assert gs == s and gw == w and gh == h
    if check_levels:
        for f, lv in enumerate(lvs):
            for l, (s, lw, lh) in enumerate(lv):
                ref = oracle.resample(frames[f], s, lw, lh)
                got = det.level_image(f, l)
                assert np.array_equal(got, ref), f"level {l} frame {f} differs"

    # ---- stage-1 scores (dense maps) and the T1 exemptions ----
    exempt1 = set()
    max_s1 = 0.0
    jobs = [(f, l) for f, lv in enumerate(lvs) for l in range(len(lv))]
    refs = _pmap(lambda fl: oracle.stage1_dense(cascade.nets[0], oracle.resample(
        frames[fl[0]], *lvs[fl[0]][fl[1]])), jobs)
    for (f, l), ref in zip(jobs, refs):
        if check_maps and ref.size:
            got = det.stage1_map(f, l).astype(np.float64)
            assert got.shape == ref.shape
            d = np.abs(got - ref)
            max_s1 = max(max_s1, float(d.max()))
            assert d.max() <= TOL, f"stage-1 map frame {f} level {l}: max err {d.max()}"
        for i, j in zip(*np.nonzero(np.abs(ref - T1) <= TOL)):
            exempt1.add((f, l, int(i), int(j)))
    rep["max_err_s1"] = max_s1
    rep["exempt_T1"] = len(exempt1)
    assert gstats["windows"] == ostats["windows"]

    # ---- survivors, selective unit, final boxes of every frame, Table-1 counts ----
    check_selective_and_boxes(gc, gboxes, gstats, ocands, oboxes, ostats, exempt1, frames, lvs,
                              cascade, T1, T2, Tnn, rule, rep=rep)
    assert rep["frames_boxes_checked"] == len(frames)
    rep["nms_frames"], rep["nms_raw"] = check_nms(gc, gboxes, len(frames))
    rep["stats"] = gstats
    if expect_exact:
        assert rep["exempt_T1"] == 0 and rep["exempt_T2"] == 0, rep
    # order of the output: (frame, score desc, y, x, w, h)
    keys = [(int(b["frame"]), -float(b["score"]), int(b["y"]), int(b["x"]), int(b["w"]), int(b["h"]))
            for b in gboxes]
    assert keys == sorted(keys)
    return rep

"""Parity helpers: compare the CUDA path (through the C ABI) with the oracle.

Bar (BASELINE.json north_star):
* pyramid levels and every integer / geometry quantity: bit-exact;
* per-window stage-1 scores and all CNN2/CNN3 responses: |gpu - oracle| <= 1e-4;
* survivor sets, K2/K3, delta, raw boxes and final boxes: exact, except windows whose
  oracle score lies within 1e-4 of T1 (and candidates with a response within 1e-4 of
  T2), which are listed and whose frames' boxes are left out of the exact comparison.
"""
import numpy as np

import oracle

TOL = 1e-4


def key(c):
    return (int(c["frame"]), int(c["level"]), int(c["iy"]), int(c["ix"]))


class Report(dict):
    pass


def oracle_maps(cascade, frames, min_face, scale_step):
    """{(frame, level): dense oracle stage-1 map} and the oracle level table."""
    lv = oracle.level_table(frames.shape[2], frames.shape[1], min_face, scale_step)
    maps = {}
    for f in range(frames.shape[0]):
        for l, (s, lw, lh) in enumerate(lv):
            maps[(f, l)] = oracle.stage1_dense(cascade.nets[0], oracle.resample(frames[f], s, lw, lh))
    return lv, maps


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


def compare_run(det, cascade, frames, min_face, scale_step, T1, T2, Tnn, rule, check_maps=True,
                check_levels=True, debug_extra=0):
    """Run the GPU detector in debug mode and the oracle on the same frames; assert parity.
    `frames`: a uint8 array (n, H, W) (ccnn_detect) or a list of 2-D frames of individual
    sizes (ccnn_detect_frames).  Returns a Report with the counts and max errors."""
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

    # ---- stage-1 scores ----
    exempt1 = set()
    max_s1 = 0.0
    if check_maps:
        for f, lv in enumerate(lvs):
            for l, (s, lw, lh) in enumerate(lv):
                ref = oracle.stage1_dense(cascade.nets[0], oracle.resample(frames[f], s, lw, lh))
                got = det.stage1_map(f, l).astype(np.float64)
                assert got.shape == ref.shape
                if ref.size:
                    d = np.abs(got - ref)
                    max_s1 = max(max_s1, float(d.max()))
                    assert d.max() <= TOL, f"stage-1 map frame {f} level {l}: max err {d.max()}"
                    for i, j in zip(*np.nonzero(np.abs(ref - T1) <= TOL)):
                        exempt1.add((f, l, int(i), int(j)))
    rep["max_err_s1"] = max_s1
    rep["exempt_T1"] = len(exempt1)

    # ---- survivor sets ----
    gmap = {key(c): c for c in gc}
    omap = {key(c): c for c in ocands}
    gset = set(gmap) - exempt1
    oset = set(omap) - exempt1
    assert gset == oset, f"survivors differ: gpu-only {sorted(gset - oset)[:5]} oracle-only {sorted(oset - gset)[:5]}"
    rep["survivors"] = len(oset)

    # ---- selective unit per common candidate ----
    bad_frames = {k[0] for k in exempt1}
    max_r = 0.0
    for k in gset:
        g, o = gmap[k], omap[k]
        assert abs(float(g["s1"]) - o["s1"]) <= TOL
        assert (g["bx"], g["by"], g["bw"], g["bh"]) == (o["bx"], o["by"], o["bw"], o["bh"])
        d2 = np.abs(g["r2"].astype(np.float64) - o["r2"])
        max_r = max(max_r, float(d2.max()))
        assert d2.max() <= TOL, f"CNN2 responses {k}: {d2.max()}"
        near2 = np.any(np.abs(o["r2"] - T2[0]) <= TOL)
        if near2:
            bad_frames.add(k[0])
            continue
        assert g["K2"] == o["K2"], k
        assert g["cnn3_ran"] == o["cnn3_ran"], k
        if o["cnn3_ran"]:
            d3 = np.abs(g["r3"].astype(np.float64) - o["r3"])
            max_r = max(max_r, float(d3.max()))
            assert d3.max() <= TOL, f"CNN3 responses {k}: {d3.max()}"
            if np.any(np.abs(o["r3"] - T2[1]) <= TOL):
                bad_frames.add(k[0])
                continue
            assert g["K3"] == o["K3"], k
        assert g["delta"] == o["delta"], k
        assert abs(float(g["score"]) - o["score"]) <= TOL
    rep["max_err_resp"] = max_r

    # ---- final boxes for frames without exemptions ----
    checked = 0
    for f in range(len(frames)):
        if f in bad_frames:
            continue
        gb = sorted((int(b["x"]), int(b["y"]), int(b["w"]), int(b["h"]), int(b["neighbors"]))
                    for b in gboxes[gboxes["frame"] == f])
        ob = sorted((int(b["x"]), int(b["y"]), int(b["w"]), int(b["h"]), int(b["neighbors"]))
                    for b in oboxes[oboxes["frame"] == f])
        assert gb == ob, f"frame {f}: boxes differ\n gpu {gb[:6]}\n ora {ob[:6]}"
        gs = np.sort(gboxes[gboxes["frame"] == f]["score"].astype(np.float64))
        os_ = np.sort(oboxes[oboxes["frame"] == f]["score"])
        assert np.all(np.abs(gs - os_) <= TOL)
        checked += 1
    rep["frames_boxes_checked"] = checked
    rep["boxes"] = len(oboxes)
    # ---- stats (Table-1 shape) ----
    assert gstats["windows"] == ostats["windows"]
    if not bad_frames and not exempt1:
        for k in ("stage1", "stage2", "stage3", "nms"):
            assert gstats[k] == ostats[k], (k, gstats[k], ostats[k])
    rep["stats"] = gstats
    # order of the output: (frame, score desc, y, x, w, h)
    keys = [(int(b["frame"]), -float(b["score"]), int(b["y"]), int(b["x"])) for b in gboxes]
    assert keys == sorted(keys)
    return rep

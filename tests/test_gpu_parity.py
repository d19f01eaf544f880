"""GPU parity: the CUDA path through the C ABI vs the oracle, element by element.

Sizes the oracle finishes in seconds that still span several stage-1 bands/segments and
ragged tails, plus BASELINE.json's full 4K size in the bench's launch configuration on
sampled outputs.  Tolerances: tests/parity.py (1e-4 absolute on scores, exact elsewhere).
"""
import numpy as np
import pytest

import oracle
from synth import arch, configs, frames as synth_frames, weights

from . import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ws():
    return weights.make_cascade_weights()


def make_det(ws, T1, T2, Tnn=2, rule=0, **kw):
    from paper_1508_01292_b200 import Detector
    args = dict(max_w=3840, max_h=2160, max_batch=32, queue_capacity=4096)
    args.update(kw)
    return Detector(arch.NETS, ws, T1, T2, Tnn, rule, **args)


def quantile_T1(cascade, frames, min_face, sf, q):
    lv, maps = parity.oracle_maps(cascade, frames, min_face, sf)
    allv = np.concatenate([m.ravel() for m in maps.values()])
    return float(np.float32(np.quantile(allv, q)))


def exact(cascade, fr, min_face, sf, q1, rule=0, Tnn=2):
    """thresholds placed on these frames with a > 1e-4 margin (tests/parity.py)."""
    T1, T2, margins = parity.exact_thresholds(cascade, fr, min_face, sf, q1, rule=rule, Tnn=Tnn)
    assert all(m is None or m > parity.TOL for m in margins), margins
    return T1, T2


def test_c1_parity_calibrated(ws, cascade):
    """The calibrated (Table-1 rate) thresholds on C1: exemptions are possible here, so every
    frame is compared against the oracle grouping with exempt decisions taken as the GPU's."""
    c = configs.C1
    T1, T2 = c.thresholds()
    fr = c.make_frames()
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    rep = parity.compare_run(det, cascade, fr, c.min_face, c.scale_step, T1, T2, c.Tnn, c.rule)
    assert rep["frames_boxes_checked"] == 1
    print(rep)


@pytest.mark.parametrize("sf", [1.05, 1.1, 1.2])
def test_c1_parity_scale_sweep(ws, cascade, sf):
    """SURVEY §8(c) coverage plan: C1 at scale_step 1.05 / 1.1 / 1.2 (45 / 23 / 12 levels incl.
    the upscaled ones) with T1 at the 1e-2 survival quantile; thresholds placed with a margin on
    the frame, so maps, survivors, K2/K3/delta, every box and the Table-1 counts are exact."""
    c = configs.C1
    fr = c.make_frames()
    T1, T2 = exact(cascade, fr, c.min_face, sf, 0.99, rule=c.rule, Tnn=c.Tnn)
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    rep = parity.compare_run(det, cascade, fr, c.min_face, sf, T1, T2, c.Tnn, c.rule,
                             expect_exact=True)
    assert rep["frames_boxes_checked"] == 1 and rep["survivors"] > 100 and rep["boxes"] > 0
    print(sf, rep)


@pytest.mark.parametrize("rule", [0, 1])
def test_c1_parity_low_threshold(ws, cascade, rule):
    """T1 near the 97% quantile so ~400 windows reach the selective unit; thresholds with a
    margin, so nothing is exempt: survivors, K2/K3/delta, final boxes and Table-1 counts are
    all exact."""
    c = configs.C1
    fr = c.make_frames()
    T1, T2 = exact(cascade, fr, c.min_face, c.scale_step, 0.97, rule=rule)
    det = make_det(ws, T1, T2, 2, rule)
    rep = parity.compare_run(det, cascade, fr, c.min_face, c.scale_step, T1, T2, 2, rule,
                             expect_exact=True)
    assert rep["survivors"] > 200 and rep["boxes"] > 0
    print(rep)


@pytest.mark.parametrize("pyr", ["tex", "ldg"])
def test_ragged_multi_frame_batch(ws, cascade, pyr):
    """odd sizes, upscaled level 0 (min_face < 27), scale 1.1, several frames per call; both
    pyramid forms (texture gathers / byte gathers)."""
    from paper_1508_01292_b200 import ccnn
    fr = synth_frames.make_stills(3, 333, 257, 991, 20)
    T1, T2 = exact(cascade, fr, 20, 1.1, 0.995, Tnn=1)
    det = make_det(ws, T1, T2, 1, 0)
    rep = parity.compare_run(det, cascade, fr, 20, 1.1, T1, T2, 1, 0,
                             debug_extra=ccnn.CCNN_DEBUG_PYR_TEX if pyr == "tex" else 0,
                             expect_exact=True)
    assert rep["boxes"] > 0
    print(rep)


def test_legacy_stage1_kernel(ws, cascade, monkeypatch):
    """The FFMA / mma.sync stage-1 kernel (stage1.cu, v8, kept as the ablation of the tcgen05
    form; selected by CCNN_S1_LEGACY=1 at ccnn_create) on the ragged multi-frame batch."""
    monkeypatch.setenv("CCNN_S1_LEGACY", "1")
    fr = synth_frames.make_stills(3, 333, 257, 991, 20)
    T1, T2 = exact(cascade, fr, 20, 1.1, 0.995, Tnn=1)
    det = make_det(ws, T1, T2, 1, 0)
    rep = parity.compare_run(det, cascade, fr, 20, 1.1, T1, T2, 1, 0, expect_exact=True)
    print(rep)


def test_fddb_like_stills(ws, cascade):
    """C2 settings (minSize 15, scaleFactor 1.05: 67 levels) on 2 of the 450x450 stills."""
    c = configs.C2
    fr = c.make_frames(2)
    T1, T2 = exact(cascade, fr, c.min_face, c.scale_step, 0.9995, Tnn=c.Tnn)
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    rep = parity.compare_run(det, cascade, fr, c.min_face, c.scale_step, T1, T2, c.Tnn, c.rule,
                             check_levels=True, expect_exact=True)
    print(rep)


def test_c4_full_size_bench_config(ws, cascade):
    """4K, min face 60, the bench's batch and launch configuration (production kernel, no
    debug map): every survivor vs the per-window oracle, sampled windows one by one vs the
    survivor set, and full oracle boxes on 2 frames."""
    c = configs.C4
    T1, T2 = c.thresholds()
    fr = c.make_frames()
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    boxes = det.detect(fr, c.min_face, c.scale_step)
    st = det.last_stats
    cands = det.candidates()
    lv = oracle.level_table(c.width, c.height, c.min_face, c.scale_step)
    assert st["windows"] == len(fr) * sum(oracle.window_grid(w, h)[0] * oracle.window_grid(w, h)[1]
                                          for _, w, h in lv)
    assert st["stage1"] == len(cands) > 0
    rng = np.random.default_rng(1)
    gset = {parity.key(x) for x in cands}
    # every survivor: per-window oracle score within 1e-4 and above T1 - 1e-4
    lev_cache = {}

    def level(f, l):
        if (f, l) not in lev_cache:
            s, w, h = lv[l]
            lev_cache[(f, l)] = oracle.resample(fr[f], s, w, h)
        return lev_cache[(f, l)]
    for x in cands:
        f, l, i, j = parity.key(x)
        s1 = oracle.stage1_window(cascade.nets[0], level(f, l), i, j)
        assert abs(float(x["s1"]) - s1) <= parity.TOL
        assert s1 > T1 - parity.TOL
    # sampled windows (uniform over frames x levels x positions) vs the survivor set
    n_checked = 0
    for _ in range(3000):
        f = int(rng.integers(len(fr)))
        l = int(rng.integers(len(lv)))
        nx, ny = oracle.window_grid(lv[l][1], lv[l][2])
        i, j = int(rng.integers(ny)), int(rng.integers(nx))
        s1 = oracle.stage1_window(cascade.nets[0], level(f, l), i, j)
        if abs(s1 - T1) <= parity.TOL:
            continue
        assert ((f, l, i, j) in gset) == (np.float32(s1) > np.float32(T1))
        n_checked += 1
    assert n_checked > 2900
    # every frame's NMS vs the oracle's grouping of the GPU's own accepted boxes (exact), and
    # the first / last frame in full vs the oracle (boxes of every frame compared, exempt
    # decisions taken as the GPU's)
    parity.check_nms(cands, boxes, len(fr))
    rep = _full_frames_vs_oracle(cascade, fr, cands, boxes, c, T1, T2, (0, len(fr) - 1))
    assert rep["frames_boxes_checked"] == 2
    print(rep)


def _full_frames_vs_oracle(cascade, fr, cands, boxes, c, T1, T2, frame_ids):
    """Survivors, selective outcome and final boxes of whole frames of a full-size batch vs
    oracle.detect of those frames (tests/parity.py check_selective_and_boxes)."""
    lv = oracle.level_table(fr.shape[2], fr.shape[1], c.min_face, c.scale_step)
    lvs = [lv] * len(fr)
    ex = parity.exempt_windows(cascade, fr, lvs, T1, frame_ids)
    rep = parity.Report()
    for f in frame_ids:
        oc, ob, _ = oracle.detect(cascade, fr[f:f + 1], c.min_face, c.scale_step, T1, T2, c.Tnn,
                                  c.rule)
        oc["frame"] = f
        ob["frame"] = f
        parity.check_selective_and_boxes(cands[cands["frame"] == f], boxes[boxes["frame"] == f],
                                         None, oc, ob, None, {k for k in ex if k[0] == f}, fr,
                                         lvs, cascade, T1, T2, c.Tnn, c.rule, frame_ids=[f],
                                         rep=rep)
    rep["exempt_T1"] = len(ex)
    return rep


def _sampled_full_size(ws, cascade, c, n_cands, n_windows, full_frames, queue_capacity=4096):
    """BASELINE config c at full size in the bench's batch and launch configuration
    (production kernels, no debug map): a sample of the survivors through the per-window
    oracle and the oracle's selective unit (score within 1e-4; K2, K3, delta exact unless a
    response lies within 1e-4 of T2; raw box exact), sampled windows one by one vs the
    survivor set, and the full oracle detection of some frames vs their boxes."""
    T1, T2 = c.thresholds()
    fr = c.make_frames()
    det = make_det(ws, T1, T2, c.Tnn, c.rule, max_w=c.width, max_h=c.height, max_batch=len(fr),
                   queue_capacity=queue_capacity)
    boxes = det.detect(fr, c.min_face, c.scale_step)
    cands = det.candidates()
    assert det.last_stats["stage1"] == len(cands) > 0
    lv = oracle.level_table(c.width, c.height, c.min_face, c.scale_step)
    params = oracle.make_params(T1, T2, c.Tnn, c.rule)
    rng = np.random.default_rng(11)
    lev_cache = {}

    def level(f, l):
        if (f, l) not in lev_cache:
            s, w, h = lv[l]
            lev_cache[(f, l)] = oracle.resample(fr[f], s, w, h)
        return lev_cache[(f, l)]
    checked_sel = 0
    for idx in rng.choice(len(cands), min(n_cands, len(cands)), replace=False):
        x = cands[idx]
        f, l, i, j = parity.key(x)
        s1 = oracle.stage1_window(cascade.nets[0], level(f, l), i, j)
        assert abs(float(x["s1"]) - s1) <= parity.TOL and s1 > T1 - parity.TOL
        assert (int(x["bx"]), int(x["by"]), int(x["bw"]), int(x["bh"])) == oracle.raw_box(lv[l][0], i, j)
        oc = oracle.classify(cascade.nets[1], cascade.nets[2], oracle.extract_patch(fr[f], lv[l][0], i, j), params)
        near = any(abs(v - T2[0]) <= parity.TOL for v in oc.r2) or \
            (oc.cnn3_ran and any(abs(v - T2[1]) <= parity.TOL for v in oc.r3))
        if near:
            continue
        assert (int(x["K2"]), int(x["K3"]), int(x["delta"]), int(x["cnn3_ran"])) == \
            (oc.K2, oc.K3, oc.delta, oc.cnn3_ran)
        assert abs(float(x["score"]) - oc.score) <= parity.TOL
        checked_sel += 1
    assert checked_sel >= 0.9 * min(n_cands, len(cands))
    gset = {parity.key(x) for x in cands}
    n_checked = 0
    for _ in range(n_windows):
        f = int(rng.integers(len(fr)))
        l = int(rng.integers(len(lv)))
        nx, ny = oracle.window_grid(lv[l][1], lv[l][2])
        i, j = int(rng.integers(ny)), int(rng.integers(nx))
        s1 = oracle.stage1_window(cascade.nets[0], level(f, l), i, j)
        if abs(s1 - T1) <= parity.TOL:
            continue
        assert ((f, l, i, j) in gset) == (np.float32(s1) > np.float32(T1))
        n_checked += 1
    assert n_checked > 0.95 * n_windows
    nf, n_raw = parity.check_nms(cands, boxes, len(fr))
    assert nf == len(fr)
    rep = _full_frames_vs_oracle(cascade, fr, cands, boxes, c, T1, T2, full_frames)
    assert rep["frames_boxes_checked"] == len(full_frames)
    print("nms raw boxes", n_raw, "full frames", rep)
    return len(cands), checked_sel


def test_c5_full_size_clutter_sampled(ws, cascade):
    """C5: 16 cluttered 4K frames at ~1% stage-1 survival (~50k survivors, the selective-unit
    and NMS stress; ~1,000 raw boxes per frame), queue capacity as in bench.py: every frame's
    NMS exact vs or_group of the GPU's accepted boxes, every frame's boxes vs oracle.detect."""
    n, k = _sampled_full_size(ws, cascade, configs.C5, 300, 2000, range(16), queue_capacity=40000)
    assert n > 10000
    print(n, k)


def test_c2_full_size_fddb_sampled(ws, cascade):
    """C2: 256 FDDB-like 450x450 stills, min face 15 (upscaled levels), scale 1.05."""
    n, k = _sampled_full_size(ws, cascade, configs.C2, 300, 3000, list(range(0, 256, 4)) + [255])
    print(n, k)


def test_c4_full_size_selective_all_survivors(ws, cascade):
    """C4 (the bench workload): every stage-1 survivor through the oracle's selective unit
    (K2, K3, delta, score, raw box), plus sampled windows and every frame's boxes vs the
    full oracle."""
    n, k = _sampled_full_size(ws, cascade, configs.C4, 100000, 2000, range(32))
    assert k >= 0.9 * n
    print(n, k)


def test_c3_full_size_1080p_sampled(ws, cascade):
    """C3: a batch of 1080p video frames, min face 40, scale 1.2."""
    n, k = _sampled_full_size(ws, cascade, configs.C3, 300, 3000, range(32))
    print(n, k)


def test_c4_debug_map_sampled(ws, cascade):
    """Dense stage-1 map of a 4K frame (debug instantiation) at 4000 sampled windows."""
    c = configs.C4
    T1, T2 = c.thresholds()
    fr = c.make_frames(2)
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    from paper_1508_01292_b200 import ccnn
    det.set_debug(ccnn.CCNN_DEBUG_STAGE1)
    det.detect(fr, c.min_face, c.scale_step)
    lv = oracle.level_table(c.width, c.height, c.min_face, c.scale_step)
    rng = np.random.default_rng(2)
    worst = 0.0
    for f in range(2):
        for l, (s, w, h) in enumerate(lv):
            L = oracle.resample(fr[f], s, w, h)
            assert np.array_equal(det.level_image(f, l), L)
            m = det.stage1_map(f, l)
            ny, nx = m.shape
            for _ in range(100):
                i, j = int(rng.integers(ny)), int(rng.integers(nx))
                d = abs(float(m[i, j]) - oracle.stage1_window(cascade.nets[0], L, i, j))
                worst = max(worst, d)
            # the last row and column of windows (ragged band / segment tails)
            for i, j in [(ny - 1, nx - 1), (0, nx - 1), (ny - 1, 0)]:
                d = abs(float(m[i, j]) - oracle.stage1_window(cascade.nets[0], L, i, j))
                worst = max(worst, d)
    assert worst <= parity.TOL, worst


def test_edge_cases(ws, cascade):
    from paper_1508_01292_b200 import ccnn
    det = make_det(ws, 0.5, (0.5, 0.5), max_w=640, max_h=480, max_batch=4, queue_capacity=64)
    # empty pyramid (frame smaller than the window at every scale): no boxes, not an error
    b = det.detect(np.zeros((1, 30, 26), np.uint8), 27, 1.2)
    assert len(b) == 0 and det.last_stats["windows"] == 0
    # exactly one window
    fr = synth_frames.make_still(27, 31, 5, 27)[None]
    det.detect(fr, 27, 1.2)
    assert det.last_stats["windows"] == 1
    # invalid arguments
    for args in [(np.zeros((1, 100, 100), np.uint8), 0, 1.2), (np.zeros((1, 100, 100), np.uint8), 24, 1.0),
                 (np.zeros((1, 500, 700), np.uint8), 24, 1.2), (np.zeros((5, 100, 100), np.uint8), 24, 1.2)]:
        with pytest.raises(ccnn.CcnnError) as e:
            det.detect(*args)
        assert e.value.code == ccnn.CCNN_E_ARG
    # survivor queue overflow is an error, never silent
    low = make_det(ws, -1.8, (0.5, 0.5), max_w=640, max_h=480, max_batch=2, queue_capacity=16)
    with pytest.raises(ccnn.CcnnError) as e:
        low.detect(configs.C1.make_frames(), 24, 1.2)
    assert e.value.code == ccnn.CCNN_E_QUEUE
    # box capacity retry semantics
    c = configs.C1
    fr = c.make_frames()
    T1 = quantile_T1(cascade, fr, c.min_face, c.scale_step, 0.97)
    d2 = make_det(ws, T1, (0.9, 0.2), max_w=640, max_h=480, max_batch=4)
    full = d2.detect(fr, c.min_face, c.scale_step)
    assert len(full) >= 1
    with pytest.raises(ccnn.CcnnError) as e:
        d2.detect(fr, c.min_face, c.scale_step, box_cap=0)
    assert e.value.code == ccnn.CCNN_E_CAPACITY


def test_8k_frame_max_size(ws, cascade):
    """A frame twice the 4K size in each dimension (7680 x 4320, min face 60: level 0 3456 x 1944,
    23 levels, 1.27 M windows): dense stage-1 maps, survivors, selective outcomes, every box and
    the Table-1 counts against the oracle, thresholds placed with a margin on the frame."""
    fr = synth_frames.make_still(7680, 4320, 8080, 60)[None]
    T1, T2 = exact(cascade, fr, 60, 1.2, 1.0 - 2e-4, Tnn=2)
    det = make_det(ws, T1, T2, 2, 0, max_w=7680, max_h=4320, max_batch=1)
    rep = parity.compare_run(det, cascade, fr, 60, 1.2, T1, T2, 2, 0, expect_exact=True)
    assert rep["frames_boxes_checked"] == 1 and rep["survivors"] > 50
    print(rep)


def test_large_batch_equals_32_frame_batches(ws):
    """96 4K frames in one call (3x the bench batch: 800 MB of frames, 526 MB of levels) give
    exactly the boxes of three 32-frame calls (frame indices offset)."""
    import torch
    c = configs.C4
    T1, T2 = c.thresholds()
    fr = torch.from_numpy(c.make_frames(96)).cuda()
    det = make_det(ws, T1, T2, c.Tnn, c.rule, max_batch=96)
    big = det.detect(fr, c.min_face, c.scale_step)
    parts = []
    for k in range(3):
        b = det.detect(fr[32 * k:32 * (k + 1)], c.min_face, c.scale_step)
        b["frame"] += 32 * k
        parts.append(b)
    assert len(big) > 0 and np.array_equal(big, np.concatenate(parts))


def test_host_vs_device_frames_and_determinism(ws):
    import torch
    c = configs.C3
    T1, T2 = c.thresholds()
    fr = c.make_frames(4)
    det = make_det(ws, T1, T2, c.Tnn, c.rule)
    a = det.detect(fr, c.min_face, c.scale_step)
    pinned = torch.from_numpy(fr).pin_memory()
    b = det.detect(pinned, c.min_face, c.scale_step)
    dev = torch.from_numpy(fr).cuda()
    d = det.detect(dev, c.min_face, c.scale_step)
    e = det.detect(dev, c.min_face, c.scale_step)
    for x in (b, d, e):
        assert np.array_equal(a, x)
    # a pitched (strided-row) device batch
    big = torch.zeros((4, c.height, c.width + 64), dtype=torch.uint8, device="cuda")
    big[:, :, :c.width] = dev
    f = det.detect(big[:, :, :c.width], c.min_face, c.scale_step)
    assert np.array_equal(a, f)
    # pitched host batches (odd pitch; pageable and pinned): the slot buffer keeps the caller's
    # pitch and the batch lands with one linear copy
    hb = torch.zeros((4, c.height, c.width + 37), dtype=torch.uint8)
    hb[:, :, :c.width] = torch.from_numpy(fr)
    assert np.array_equal(a, det.detect(hb[:, :, :c.width], c.min_face, c.scale_step))
    assert np.array_equal(a, det.detect(hb.pin_memory()[:, :, :c.width], c.min_face, c.scale_step))


def test_host_frames_odd_width_linear_copy(ws, cascade):
    """C2-like stills of odd width (450: rows not 16-B aligned) from host memory, contiguous
    (one linear H2D of the whole batch, device pitch 450) and pinned, equal the device-resident
    detection and the oracle's levels."""
    import torch
    from paper_1508_01292_b200 import ccnn
    fr = synth_frames.make_stills(6, 450, 451, 77, 15)
    T1, T2 = configs.C2.thresholds()
    det = make_det(ws, T1, T2, configs.C2.Tnn, configs.C2.rule, max_w=450, max_h=451, max_batch=8)
    ref = det.detect(torch.from_numpy(fr).cuda(), 15, 1.05)
    det.set_debug(ccnn.CCNN_DEBUG_LEVELS)
    assert np.array_equal(det.detect(fr, 15, 1.05), ref)
    lv = oracle.level_table(450, 451, 15, 1.05)
    for f in (0, 5):
        for l in (0, len(lv) // 2, len(lv) - 1):
            s, lw, lh = lv[l]
            assert np.array_equal(det.level_image(f, l), oracle.resample(fr[f], s, lw, lh))
    assert np.array_equal(det.detect(torch.from_numpy(fr).pin_memory(), 15, 1.05), ref)
    assert len(ref) > 0


def test_streaming_submit_collect(ws):
    """ccnn_submit / ccnn_collect (two batches in flight, H2D overlapped) returns exactly what
    ccnn_detect returns, in submission order; the in-flight limit and detect-while-in-flight
    are errors."""
    import torch
    from paper_1508_01292_b200 import ccnn
    c = configs.C3
    T1, T2 = c.thresholds()
    batches = [c.make_frames(3, seed=configs.FRAME_SEED + 11 * k) for k in range(4)]
    det = make_det(ws, T1, T2, c.Tnn, c.rule, max_batch=4)
    ref = [det.detect(b, c.min_face, c.scale_step) for b in batches]
    pinned = [torch.from_numpy(b).pin_memory() for b in batches]
    got = []
    for k, b in enumerate(pinned):
        det.submit(b, c.min_face, c.scale_step)
        if k:
            got.append(det.collect())
    with pytest.raises(ccnn.CcnnError) as e:         # one in flight: detect is refused
        det.detect(batches[0], c.min_face, c.scale_step)
    assert e.value.code == ccnn.CCNN_E_STATE
    det.submit(pinned[0], c.min_face, c.scale_step)
    det.submit(pinned[1], c.min_face, c.scale_step)     # three in flight
    with pytest.raises(ccnn.CcnnError) as e:         # a fourth batch is refused
        det.submit(pinned[2], c.min_face, c.scale_step)
    assert e.value.code == ccnn.CCNN_E_STATE
    got.append(det.collect())
    got.append(det.collect())
    got.append(det.collect())
    for k in range(4):
        assert np.array_equal(got[k], ref[k])
    assert np.array_equal(got[4], ref[0])
    assert np.array_equal(got[5], ref[1])


def test_streaming_device_frames_overlapped_pyramid(ws, cascade):
    """The bench's path: device-resident batches, three in flight, so batch k+2's pyramid (own
    stream, own level arena) overlaps batch k's stage 1 .. NMS.  Every collected batch equals
    oracle.detect of its frames (survivors, selective outcome, every frame's boxes, Table-1
    counts; thresholds placed with a margin on these frames, so nothing is exempt) and the
    synchronous ccnn_detect of the same batch (C4 4K frames, distinct content per batch;
    P:127 "CNN1 moves to the next level regardless", S:426 mode equivalence)."""
    import torch
    c = configs.C4
    host = [c.make_frames(3, seed=configs.FRAME_SEED + 13 * k) for k in range(5)]
    allf = np.concatenate(host)
    T1, T2 = exact(cascade, allf, c.min_face, c.scale_step, 1.0 - 2e-4, Tnn=c.Tnn)
    batches = [torch.from_numpy(h).cuda() for h in host]
    det = make_det(ws, T1, T2, c.Tnn, c.rule, max_batch=4)
    got = []

    def collect():
        b = det.collect()
        got.append((b, det.candidates(), dict(det.last_stats)))
    det.submit(batches[0], c.min_face, c.scale_step)
    det.submit(batches[1], c.min_face, c.scale_step)
    for k in range(2, len(batches)):                  # three in flight
        det.submit(batches[k], c.min_face, c.scale_step)
        collect()
    collect()
    collect()
    lv = oracle.level_table(c.width, c.height, c.min_face, c.scale_step)
    total = 0
    for k, (gb, gc, gst) in enumerate(got):
        fr = host[k]
        oc, ob, ost = oracle.detect(cascade, fr, c.min_face, c.scale_step, T1, T2, c.Tnn, c.rule)
        ex = parity.exempt_windows(cascade, fr, [lv] * len(fr), T1)
        assert not ex
        rep = parity.check_selective_and_boxes(gc, gb, gst, oc, ob, ost, ex, fr, [lv] * len(fr),
                                               cascade, T1, T2, c.Tnn, c.rule)
        assert rep["frames_boxes_checked"] == len(fr) and rep["exempt_T2"] == 0, rep
        parity.check_nms(gc, gb, len(fr))
        assert np.array_equal(gb, det.detect(batches[k], c.min_face, c.scale_step)), k
        total += len(gb)
        print(k, rep)
    assert total > 0


@pytest.mark.parametrize("seg", [1, 3, 7])
def test_segment_heights_and_patchwork(ws, cascade, seg):
    """Forced short segments (every task boundary, priming and ring wrap-around) and
    patchwork bands (many narrow levels of a 1080p frame packed side by side): the dense
    stage-1 maps and survivors still match the oracle."""
    c = configs.C3
    fr = c.make_frames(1)
    T1, T2 = exact(cascade, fr, 96, 1.25, 0.999)
    det = make_det(ws, T1, T2, 2, 0, max_batch=2, segment_rows=seg)
    rep = parity.compare_run(det, cascade, fr, 96, 1.25, T1, T2, 2, 0, check_levels=False,
                             expect_exact=True)
    assert rep["survivors"] > 10
    print(rep)


def _quantile_T1_list(cascade, frames, min_face, sf, q):
    vals = []
    for fr in frames:
        _, maps = parity.oracle_maps(cascade, fr[None], min_face, sf)
        vals += [m.ravel() for m in maps.values()]
    return float(np.float32(np.quantile(np.concatenate(vals), q)))


def _mixed_frames():
    """stills of individual sizes in one call, including a frame
    with an empty pyramid in the middle and a 1-pixel-wide one at the end."""
    return [synth_frames.make_still(333, 257, 991, 20), synth_frames.make_still(450, 450, 992, 20),
            np.random.default_rng(993).integers(0, 256, (30, 26), dtype=np.uint8), synth_frames.make_still(320, 240, 994, 20),
            synth_frames.make_still(97, 131, 995, 20), np.full((40, 1), 77, np.uint8)]


def test_mixed_size_frames_parity(ws, cascade):
    fr = _mixed_frames()
    T1, T2 = exact(cascade, fr, 20, 1.15, 0.995, Tnn=1)
    det = make_det(ws, T1, T2, 1, 0, max_w=640, max_h=480, max_batch=8)
    rep = parity.compare_run(det, cascade, fr, 20, 1.15, T1, T2, 1, 0, expect_exact=True)
    assert rep["survivors"] > 50 and rep["frames_boxes_checked"] == len(fr)
    print(rep)


def test_mixed_size_frames_api(ws, cascade):
    """detect_frames == one detect per frame; host, pinned, device and pitched device frames
    agree; submit_frames interleaves with submit; replans between shapes are exact."""
    import torch
    fr = _mixed_frames()
    T1, T2 = _quantile_T1_list(cascade, fr, 20, 1.15, 0.99), (0.8, 0.1)
    det = make_det(ws, T1, T2, 1, 0, max_w=640, max_h=480, max_batch=8)
    per = []
    for f, x in enumerate(fr):
        b = det.detect(x[None], 20, 1.15)
        b["frame"] = f
        per.append(b)
    ref = np.concatenate(per)
    a = det.detect_frames(fr, 20, 1.15)
    assert np.array_equal(a, ref)
    pinned = [torch.from_numpy(x).pin_memory() for x in fr]
    assert np.array_equal(det.detect_frames(pinned, 20, 1.15), ref)
    dev = []
    for x in fr:                                       # pitched device views
        big = torch.zeros((x.shape[0], x.shape[1] + 37), dtype=torch.uint8, device="cuda")
        big[:, :x.shape[1]] = torch.from_numpy(x).cuda()
        dev.append(big[:, :x.shape[1]])
    assert np.array_equal(det.detect_frames(dev, 20, 1.15), ref)
    # streaming: alternate frame lists and uniform batches, two in flight
    uni = np.stack([fr[0], fr[0]])
    det.submit_frames(pinned, 20, 1.15)
    det.submit(uni, 20, 1.15)
    g0 = det.collect()
    det.submit_frames(fr[::-1], 20, 1.15)
    g1 = det.collect()
    g2 = det.collect()
    assert np.array_equal(g0, ref)
    u = det.detect(uni, 20, 1.15)
    assert np.array_equal(g1, u)
    rev = np.concatenate([per[len(fr) - 1 - k] for k in range(len(fr))])
    rev["frame"] = np.repeat(np.arange(len(fr)), [len(per[len(fr) - 1 - k]) for k in range(len(fr))])
    assert np.array_equal(g2, rev)


def test_synthetic_gt_scores_match_oracle(ws, cascade):
    """NEXT #3: FDDB / AFW protocol scores of the CUDA path's boxes on planted-face stills of
    mixed sizes equal the scores of the oracle's boxes (evaluate.py is host-side scoring)."""
    from paper_1508_01292_b200 import evaluate as ev
    data = [synth_frames.make_still_gt(w, h, 500 + k, 15, n_faces=4)
            for k, (w, h) in enumerate([(300, 260), (450, 450), (380, 290), (257, 333)])]
    fr = [d[0] for d in data]
    T1 = _quantile_T1_list(cascade, fr, 15, 1.05, 0.998)
    T2 = (0.5, 0.0)
    det = make_det(ws, T1, T2, 1, 0, max_w=512, max_h=512, max_batch=8, queue_capacity=8192)
    g = det.detect_frames(fr, 15, 1.05)
    _, o, _ = parity._oracle_frames(cascade, fr, 15, 1.05, T1, T2, 1, 0)
    assert len(g) > 0
    gp, op = ev.boxes_by_frame(g, len(fr)), ev.boxes_by_frame(o, len(fr))
    ths = [-2.0, 0.0, 0.5]
    # same boxes; scores within 1e-4 and none near these thresholds -> identical ROC rows
    assert ev.score_fddb([(d[1], p[0], p[1]) for d, p in zip(data, gp)], ths) == \
        ev.score_fddb([(d[1], p[0], p[1]) for d, p in zip(data, op)], ths)
    assert ev.score_afw([(d[1], p[0]) for d, p in zip(data, gp)]) == \
        ev.score_afw([(d[1], p[0]) for d, p in zip(data, op)])


def test_rgb_ingest(ws, cascade):
    """Interleaved R,G,B frames (host, pinned, device, pitched device; mixed with gray frames
    in one batch) give exactly the boxes and pyramid levels of their oracle Rec.601 gray
    planes (reading I1)."""
    import torch
    from paper_1508_01292_b200 import ccnn
    rng = np.random.default_rng(21)
    grays = [synth_frames.make_still(w, h, 300 + k, 20) for k, (w, h) in
             enumerate([(333, 257), (320, 240), (201, 150)])]
    # colourise: R,G,B planes that are not a function of the gray value alone
    rgbs = [np.stack([g, np.clip(g.astype(int) + rng.integers(-40, 41, g.shape), 0, 255),
                      rng.integers(0, 256, g.shape)], 2).astype(np.uint8) for g in grays]
    ref_gray = [oracle.to_gray(x) for x in rgbs]
    mixed = [rgbs[0], grays[1], rgbs[2]]
    mixed_gray = [ref_gray[0], grays[1], ref_gray[2]]
    T1 = _quantile_T1_list(cascade, mixed_gray, 20, 1.15, 0.995)
    det = make_det(ws, T1, (0.8, 0.1), 1, 0, max_w=640, max_h=480, max_batch=8)
    ref = det.detect_frames(mixed_gray, 20, 1.15)
    det.set_debug(ccnn.CCNN_DEBUG_LEVELS)
    got = det.detect_frames(mixed, 20, 1.15)
    assert np.array_equal(got, ref)
    # pyramid (gather and 4-column classes: here min face 20 < 27, so level 0 is upscaled and
    # both occur), stage 1, selective CNN2 (tcgen05) and CNN3 + rule, NMS, plus one R,G,B -> gray
    # conversion
    assert det.last_stats["kernel_launches"] == 7
    for f in (0, 2):
        for l, (s, lw, lh) in enumerate(oracle.level_table(mixed[f].shape[1], mixed[f].shape[0], 20, 1.15)[:3]):
            assert np.array_equal(det.level_image(f, l), oracle.resample(mixed_gray[f], s, lw, lh))
    pinned = [torch.from_numpy(x).pin_memory() for x in mixed]
    assert np.array_equal(det.detect_frames(pinned, 20, 1.15), ref)
    dev = [torch.from_numpy(x).cuda() for x in mixed]
    assert np.array_equal(det.detect_frames(dev, 20, 1.15), ref)
    pitched = []
    for x in mixed:                                     # odd row pitch on the device
        big = torch.zeros((x.shape[0], x.shape[1] + 7) + x.shape[2:], dtype=torch.uint8, device="cuda")
        big[:, :x.shape[1]] = torch.from_numpy(x).cuda()
        pitched.append(big[:, :x.shape[1]])
    assert np.array_equal(det.detect_frames(pitched, 20, 1.15), ref)
    # streaming with RGB
    det.submit_frames(pinned, 20, 1.15)
    det.submit_frames(dev, 20, 1.15)
    assert np.array_equal(det.collect(), ref)
    assert np.array_equal(det.collect(), ref)
    # bad channel counts are argument errors
    with pytest.raises(ccnn.CcnnError) as e:
        det.detect_frames([np.zeros((40, 40, 2), np.uint8)], 20, 1.15)
    assert e.value.code == ccnn.CCNN_E_ARG


def test_fp32_ffma_vs_split_fp16_tcgen05_precision(ws, cascade, monkeypatch):
    """north_star names an fp32 FMA path for stage 1; the product kernel runs the three conv
    layers as fp16 hi+lo split tcgen05 MMAs with fp32 accumulation.  Side by side on the same
    frames (two 1080p frames, every window of every level): both kernels' dense stage-1 maps
    against the fp64 oracle, and against each other.  Both must meet the 1e-4 bar; the split
    form's error is reported (profiles/r2_precision.txt records a run)."""
    from paper_1508_01292_b200 import ccnn
    c = configs.C3
    fr = c.make_frames(2)
    T1, T2 = c.thresholds()
    lv, maps = parity.oracle_maps(cascade, fr, c.min_face, c.scale_step)
    got = {}
    for legacy in ("0", "1"):
        monkeypatch.setenv("CCNN_S1_LEGACY", legacy)
        det = make_det(ws, T1, T2, c.Tnn, c.rule, max_batch=2)
        det.set_debug(ccnn.CCNN_DEBUG_STAGE1)
        det.detect(fr, c.min_face, c.scale_step)
        got[legacy] = {k: det.stage1_map(*k).astype(np.float64) for k in maps}
        det.close()
    err = {}
    for legacy in ("0", "1"):
        err[legacy] = max(float(np.max(np.abs(got[legacy][k] - maps[k]))) for k in maps if maps[k].size)
    between = max(float(np.max(np.abs(got["0"][k] - got["1"][k]))) for k in maps if maps[k].size)
    n = sum(m.size for m in maps.values())
    print(f"windows {n}: max |tcgen05 split-fp16 - fp64 oracle| = {err['0']:.3e}, "
          f"max |FFMA fp32 - fp64 oracle| = {err['1']:.3e}, max |tcgen05 - FFMA| = {between:.3e}")
    assert err["0"] <= parity.TOL and err["1"] <= parity.TOL

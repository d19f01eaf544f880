"""bench.py -- 4K UHD frames/s (min face 60 px) and stage-1 Gwindows/s of the B200 hot path.

Contract:
  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c4]
  N > 1: one rank per GPU (under torchrun, or spawned by bench.py itself through
  torch.distributed.run when WORLD_SIZE is unset); the global stream of N x batch frames is
  sharded by frame (rank r owns frames g = r mod N: weak scaling); the only collective is
  the final all_gather of the detections (NCCL; gloo when ranks share a GPU, e.g.
  --dist-backend gloo on a 1-GPU box), and rank 0 checks the merged boxes bit for bit
  against a 1-rank detection of the same global frames.
A step = one batch of synthetic frames through the public API (ccnn_submit + ccnn_collect,
three batches in flight; pyramid -> fused stage 1 -> selective unit -> NMS -> boxes on the host).  `value` is timed with CUDA events on the
ctx stream with the batch already resident in HBM (265 MB of 4K frames per step, larger
than the 126 MB L2); `e2e` is the same call with the frames in pinned HOST memory
(H2D inside the timed region).  Rank 0 prints ONE JSON line.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_4K_FPS = 27.0   # PAPER.md P:17 / P:245-255 (mobile Kepler + Ivy Bridge): context


def stage1_alg_flops(levels):
    """Algorithmic stage-1 FLOPs of one frame: 2 x MACs of the dense fully-convolutional
    CNN1 over the conv outputs some window needs."""
    tot = 0
    for _, lw, lh in levels:
        nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
        macs = ((4 * nx + 20) * (4 * ny + 24) * 6 * 16      # C4x4 1->6
                + (2 * nx + 8) * (2 * ny + 10) * 6 * 54      # C3x3 6->6
                + nx * ny * (2 * 180 + 2))                   # C5x6 6->2, C1x1 2->1
        tot += 2 * macs
    return tot


def split_mma_factor(levels):
    """MMAs per fp32-accurate product in stage 1, weighted by the layers' algorithmic FLOPs:
    layer 1 multiplies exact fp16 pixels by hi + lo weights (2 MMAs), layers 2-3 split both
    operands (hi*hi + hi*lo + lo*hi: 3 MMAs); layer 4 (1x1) runs on the FFMA pipe and counts
    at 3 like its layer-3 neighbour (it is 0.5% of the work)."""
    l1 = l23 = 0
    for _, lw, lh in levels:
        nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
        l1 += (4 * nx + 20) * (4 * ny + 24) * 6 * 16
        l23 += (2 * nx + 8) * (2 * ny + 10) * 6 * 54 + nx * ny * (2 * 180 + 2)
    return (2.0 * l1 + 3.0 * l23) / (l1 + l23) if l1 + l23 else 3.0


def level_table(W, H, min_face, sf):
    """Level sizes for reporting (same O1 rule as the library; floats only for counting)."""
    out = []
    s = 27.0 / min_face
    sfd = float(np.float32(sf))
    while True:
        lw, lh = int(np.floor(W * s)), int(np.floor(H * s))
        if lw < 27 or lh < 31:
            break
        out.append((s, lw, lh))
        s = s / sfd
    return out


class ClockSampler:
    """SM clocks / throttle reasons sampled every 20 ms by an in-process NVML thread (cheap
    calls, no driver-lock contention with the measured work) while
    the GPU is under load: only the samples between mark_load() and stop() are reported (all,
    if none)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []                  # (time, sm_mhz, max_mhz, set of reasons)
        self.t_load = None
        self.stop_ev = threading.Event()
        self.thread = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(self.index).uuid)
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def run():
                while not self.stop_ev.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((time.perf_counter(), float(sm), float(mx),
                                          {n for n, bit in zip(self.NAMES, bits) if r & bit}))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.02)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None

    def mark_load(self):
        self.t_load = time.perf_counter()

    def stop(self):
        t_end = time.perf_counter()
        self.stop_ev.set()
        if self.thread:
            self.thread.join(1.0)
        if not self.rows:
            return None
        rows = [r for r in self.rows if self.t_load is not None and self.t_load <= r[0] <= t_end]
        window = "load" if rows else "all"
        rows = rows or self.rows
        return {"sm_mhz": float(np.median([r[1] for r in rows])), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": sorted(set().union(*[r[3] for r in rows])), "samples": len(rows),
                "window": window, "source": "nvml"}


def parse_cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def bind_host_to_gpu(dev_index):
    """Pin this process to the CPUs of the GPU's NUMA node (so the pinned host frames are
    allocated on the node whose PCIe root hosts the GPU: the H2D of e2e then does not cross the
    socket interconnect).  Returns (previous affinity or None, outcome text)."""
    try:
        import torch
        # the PCI address from the CUDA device properties, not an nvidia-smi subprocess: a
        # driver query from another process right before the e2e loop was measured to slow
        # the loop's H2D copies (tools/e2e_probe.py: 6.6k -> 4.5k frames/s at C4)
        p = torch.cuda.get_device_properties(dev_index)
        bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            cpus = parse_cpulist(f.read())
        old = os.sched_getaffinity(0)
        use = cpus & old
        if not use:
            return None, f"not bound: GPU {bus} local CPUs outside this process's affinity"
        if use == old:
            return None, f"not bound: all {len(old)} usable CPUs are local to GPU {bus}"
        os.sched_setaffinity(0, use)
        return old, f"bound to the {len(use)} CPUs local to GPU {bus}"
    except Exception as e:
        return None, f"not bound: topology unknown ({type(e).__name__})"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, cascade_ws, frames, T1, T2, budget_s=10.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload
    (SURVEY §8(d)): the dense-scan oracle on all cores (`value`), on 1 core, and the
    per-window oracle (the plain definition) on all cores (one 4K frame) and on 1 core
    (one C1 320x240 frame: windows/s)."""
    import oracle
    from synth import arch, configs
    cas = oracle.Cascade(arch.NETS, cascade_ws)
    cores = len(os.sched_getaffinity(0))

    def run(frs, dense, threads, c=cfg, budget=None):
        t0 = time.perf_counter()
        n = 0
        while n < len(frs):
            oracle.detect(cas, frs[n:n + 1], c.min_face, c.scale_step, T1, T2, c.Tnn, c.rule,
                          dense=dense, n_threads=threads)
            n += 1
            if budget is None or time.perf_counter() - t0 > budget:
                break
        return n, time.perf_counter() - t0

    n, dt = run(frames, True, cores, budget=budget_s)
    n1, dt1 = run(frames, True, 1)
    npw, dtpw = run(frames, False, cores)
    c1 = configs.C1
    f1 = c1.make_frames(1)
    lv1 = oracle.level_table(c1.width, c1.height, c1.min_face, c1.scale_step)
    w1 = sum(oracle.window_grid(w, h)[0] * oracle.window_grid(w, h)[1] for _, w, h in lv1)
    _, dtc1 = run(f1, False, 1, c=c1)
    wpf = sum(((w - 27) // 4 + 1) * ((h - 31) // 4 + 1) for _, w, h in level_table(
        cfg.width, cfg.height, cfg.min_face, cfg.scale_step))
    return {"value": n / dt, "unit": "frames/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{n} of the bench's {cfg.width}x{cfg.height} frames through oracle.detect "
                      f"(C, fp64, dense stage-1 scan, {cores} threads), {dt:.1f} s",
            "dense_1core": {"value": n1 / dt1, "unit": "frames/s", "cores": 1,
                            "windows_per_s": wpf * n1 / dt1, "sample": f"{n1} frame, {dt1:.1f} s"},
            "per_window_all_cores": {"value": npw / dtpw, "unit": "frames/s", "cores": cores,
                                     "windows_per_s": wpf * npw / dtpw,
                                     "sample": f"{npw} frame, per-window CNN1 (dense=False), {dtpw:.1f} s"},
            "per_window_1core_c1": {"value": 1.0 / dtc1, "unit": "frames/s", "cores": 1,
                                    "windows_per_s": w1 / dtc1,
                                    "sample": f"1 C1 320x240 frame (min face 24), per-window, {dtc1:.1f} s"}}


def ncu_stage1_traffic(cfg_id, batch, seg, timeout=240):
    """DRAM bytes read + written by ONE stage-1 launch of this workload, measured now by an ncu
    pass over a probe run of this script (None if ncu is unavailable or fails)."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--print-units", "base", "-k", "regex:stage1_tc", "-s", "2",
           "-c", "1", "--csv", sys.executable, os.path.abspath(__file__), "--probe", "--config",
           cfg_id, "--batch", str(batch), "--seg", str(seg)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
        rows = list(csv.reader(io.StringIO(out[out.index('"ID"'):])))
        hdr = rows[0]
        iname, ival = hdr.index("Metric Name"), hdr.index("Metric Value")
        m = {r[iname]: float(r[ival].replace(",", "")) for r in rows[1:] if len(r) > ival}
        return m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"], \
            "ncu live (dram__bytes_read.sum + dram__bytes_write.sum, one launch, %.3f ms)" % (
                m.get("gpu__time_duration.sum", 0.0) / 1e6)
    except Exception as e:
        return None, "ncu probe failed: %s" % type(e).__name__


def probe(args, cfg):
    """--probe: a few synchronous detects of the workload (the ncu traffic pass runs this)."""
    import torch
    from paper_1508_01292_b200 import Detector
    from synth import arch, weights
    T1, T2 = cfg.thresholds()
    batch = args.batch or cfg.batch
    det = Detector(arch.NETS, weights.make_cascade_weights(), T1, T2, cfg.Tnn, cfg.rule,
                   max_w=cfg.width, max_h=cfg.height, max_batch=batch,
                   queue_capacity=40000 if cfg.kind == "clutter" else 4096, segment_rows=args.seg)
    fr = torch.from_numpy(cfg.make_frames(batch)).cuda()
    for _ in range(4):
        det.detect(fr, cfg.min_face, cfg.scale_step)
    det.close()
    return 0


def run_reference(args, cfg):
    """--impl reference: the oracle (the only reference this tier has), on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import weights
    ws = weights.make_cascade_weights()
    T1, T2 = cfg.thresholds()
    frames = cfg.make_frames(max(1, args.warmup + args.steps))
    import oracle
    from synth import arch
    cas = oracle.Cascade(arch.NETS, ws)
    cores = len(os.sched_getaffinity(0))
    for k in range(min(args.warmup, 1)):      # the oracle has no warm-up effects worth more
        oracle.detect(cas, frames[k:k + 1], cfg.min_face, cfg.scale_step, T1, T2, cfg.Tnn, cfg.rule)
    t0 = time.perf_counter()
    for k in range(args.steps):
        f = args.warmup + k
        oracle.detect(cas, frames[f:f + 1], cfg.min_face, cfg.scale_step, T1, T2, cfg.Tnn, cfg.rule)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": "4K UHD frames/s (min face 60px)", "value": v,
            "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": v / PAPER_4K_FPS, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "frames_per_step_per_gpu": cfg.batch, "W": cfg.width,
                       "H": cfg.height, "min_face": cfg.min_face, "scale_step": cfg.scale_step,
                       "Tnn": cfg.Tnn, "sample": "1 frame of the workload per step"},
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": f"1 frame per step of {cfg.name} through oracle.detect "
                                       f"(C, fp64, dense stage-1 scan, {cores} threads)"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: launch N ranks of this script through
    torch.distributed.run on this node (127.0.0.1), pass rank 0's output through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--batch", type=int, default=0, help="frames per step per GPU (0 = config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-traffic", action="store_true", help="skip the live ncu traffic pass")
    ap.add_argument("--no-verify-merge", action="store_true")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="auto: nccl with one GPU per rank, gloo when ranks share GPUs")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--seg", type=int, default=0, help="stage-1 segment rows (0 = adaptive)")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from synth import configs, weights
    cfg = configs.BY_ID[args.config]
    if args.probe:
        return probe(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    n_dev = torch.cuda.device_count()
    dist, backend = None, None
    torch.cuda.set_device(local % n_dev)
    dev = torch.device("cuda", torch.cuda.current_device())
    if world > 1:
        import torch.distributed as dist
        backend = args.dist_backend
        if backend == "auto":
            backend = "nccl" if n_dev >= world else "gloo"
        if backend == "nccl" and n_dev < world:
            print(f"bench.py: {world} NCCL ranks need {world} GPUs ({n_dev} visible); "
                  "use --dist-backend gloo to share GPUs", file=sys.stderr)
            return 2
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    coll_dev = dev if backend == "nccl" else torch.device("cpu")

    from paper_1508_01292_b200 import Detector
    from paper_1508_01292_b200 import dist as cdist
    from synth import arch
    ws = weights.make_cascade_weights()
    T1, T2 = cfg.thresholds()
    batch = args.batch or cfg.batch
    # frame-sharded weak scaling: the global stream has world x batch frames; rank r owns the
    # frames g = r mod world (frames are independent, BASELINE north_star)
    n_global = world * batch
    my_ids = cdist.shard_frames(n_global, world, rank)
    frames = cfg.make_frames_at(my_ids, n_global)
    det = Detector(arch.NETS, ws, T1, T2, cfg.Tnn, cfg.rule, max_w=cfg.width, max_h=cfg.height,
                   max_batch=batch, queue_capacity=max(4096, 40000 if cfg.kind == "clutter" else 0),
                   segment_rows=args.seg, device=dev.index)
    stream = torch.cuda.current_stream(dev)
    det.set_stream(stream.cuda_stream)
    dframes = torch.from_numpy(frames).to(dev)
    levels = level_table(cfg.width, cfg.height, cfg.min_face, cfg.scale_step)
    windows_per_frame = sum(((w - 27) // 4 + 1) * ((h - 31) // 4 + 1) for _, w, h in levels)
    flops_per_frame = stage1_alg_flops(levels)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        det.detect(dframes, cfg.min_face, cfg.scale_step)
    clocks = ClockSampler(dev.index) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    barrier()
    if clocks:
        clocks.mark_load()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s1_ms, launches, all_boxes, mma_flops = 0.0, 0, [], 0.0
    stats = None
    # the streaming public API (ccnn_submit / ccnn_collect) with three batches in flight: batch
    # k+2 is enqueued before batch k's boxes are collected, so the host's per-call work, the D2H
    # of the boxes and the next batches' pyramids overlap the device work (each step still
    # produces its boxes on the host)
    e0.record(stream)
    for k in range(min(2, args.steps)):
        det.submit(dframes, cfg.min_face, cfg.scale_step)
    for k in range(args.steps):
        if k + 2 < args.steps:
            det.submit(dframes, cfg.min_face, cfg.scale_step)
        b = det.collect()
        stats = det.last_stats
        s1_ms += stats["ms"][2]
        mma_flops += stats["s1_mma_flops"]
        launches += stats["kernel_launches"]
        all_boxes.append(b)
    # the only cross-GPU exchange: gather every rank's detections, once
    merged = None
    if dist is not None:
        merged = cdist.gather_boxes(cdist.to_global(all_boxes[-1], my_ids),
                                    device=dev if backend == "nccl" else None)
    e1.record(stream)
    e1.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))

    # ---- e2e: the streaming public API (ccnn_submit / ccnn_collect) with the frames in
    #      pinned HOST memory: every step copies its frames H2D and reads its boxes back;
    #      the copy of step k+1 overlaps the kernels of step k (three batches in flight) ----
    # enough steps for a >= ~300 ms e2e region (host jitter of a few ms must not dominate a
    # small config's rate): estimate a step from the device-timed loop + H2D at ~40 GB/s
    est_ms = ms / args.steps + frames.nbytes / 40e9 * 1e3
    e2e_steps = args.e2e_steps or int(min(2000, max(10, args.steps, np.ceil(300.0 / max(est_ms, 1e-3)))))
    # per-stage device times of synchronous calls (no neighbouring batches on the GPU): what
    # each kernel costs alone, e.g. the pyramid's bandwidth (outside the timed regions)
    alone = []
    for _ in range(3):
        det.detect(dframes, cfg.min_face, cfg.scale_step)
        alone.append(det.last_stats["ms"])
    alone = [float(x) for x in np.median(np.array(alone), axis=0)]
    old_aff, numa = bind_host_to_gpu(dev.index)
    host = torch.from_numpy(frames).pin_memory()
    det.detect(host, cfg.min_face, cfg.scale_step)
    barrier()
    t_e2e0 = time.perf_counter()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    d2h = 0
    for k in range(min(2, e2e_steps)):
        det.submit(host, cfg.min_face, cfg.scale_step, timed=False)
    for k in range(e2e_steps):
        if k + 2 < e2e_steps:
            det.submit(host, cfg.min_face, cfg.scale_step, timed=False)
        d2h += det.collect().nbytes + 64
    h1.record(stream)
    h1.synchronize()
    barrier()
    ms_e2e = max_over_ranks(max(h0.elapsed_time(h1), 1000.0 * (time.perf_counter() - t_e2e0) - 1.0))
    clk = clocks.stop() if clocks else None     # device-timed + e2e regions (both under load)
    # pure H2D rate of these pinned frames on this box (the e2e path's bound at 4K)
    hbuf = torch.empty_like(dframes)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(3):
        hbuf.copy_(host, non_blocking=True)
    c1.record(stream)
    c1.synchronize()
    h2d_gbs = 3 * frames.nbytes / (c0.elapsed_time(c1) / 1000.0) / 1e9
    del hbuf
    if old_aff is not None:
        os.sched_setaffinity(0, old_aff)

    # ---- batch-1 latency: one frame per synchronous ccnn_detect (device-resident frame) ----
    lat_wall, lat_dev = [], []
    one = dframes[:1]
    for k in range(23):
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        q0.record(stream)
        det.detect(one, cfg.min_face, cfg.scale_step)
        q1.record(stream)
        q1.synchronize()
        if k >= 3:
            lat_wall.append(1000.0 * (time.perf_counter() - t0))
            lat_dev.append(q0.elapsed_time(q1))

    # ---- merged detections vs a 1-rank run over the same global frames (bit for bit) ----
    merge_check = None
    if dist is not None and not args.no_verify_merge:
        ok = None
        if rank == 0:
            ref = []
            for g0 in range(0, n_global, batch):
                ids = np.arange(g0, min(n_global, g0 + batch))
                fr = torch.from_numpy(cfg.make_frames_at(ids, n_global)).to(dev)
                ref.append(cdist.to_global(det.detect(fr, cfg.min_face, cfg.scale_step), ids))
            ref = cdist.sort_boxes(np.concatenate(ref))
            ok = bool(len(ref) == len(merged) and ref.tobytes() == merged.tobytes())
            merge_check = {"global_frames": n_global, "merged_boxes": int(len(merged)),
                           "reference": "1-rank ccnn_detect of the same global frames on rank 0",
                           "bit_exact": ok}
        barrier()

    traffic, traffic_src = None, "not measured (--no-traffic)"
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic, traffic_src = ncu_stage1_traffic(args.config, batch, args.seg)

    if rank == 0:
        total_frames = world * batch * args.steps
        value = total_frames / (ms / 1000.0)
        s1_avg_ms = s1_ms / args.steps
        achieved_tflops = flops_per_frame * batch / (s1_avg_ms / 1000.0) / 1e12
        peaks = measured_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12     # FFMA pipe peak
        # stage 1 runs its three conv layers as fp16 tcgen05 MMAs (exact pixels, hi+lo split
        # weights / activations, fp32 accumulators): the dense fp16 tensor peak binds.  The
        # timed region is short (~15 ms) and runs at the max SM clock (clocks below), so the
        # burst figure applies (bf16 and fp16 share the nominal rate, B200_PROFILING.md)
        tc_peak = float(peaks.get("bf16_tflops", 2250.0))
        line = {
            "metric": "4K UHD frames/s (min face 60px)",
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": value / PAPER_4K_FPS, "dtype": "f16*f16->f32 (hi+lo split MMAs, f32 epilogues)",
            "data": "synthetic",
            "config": {"workload": cfg.name, "frames_per_step_per_gpu": batch, "W": cfg.width,
                       "H": cfg.height, "min_face": cfg.min_face, "scale_step": cfg.scale_step,
                       "Tnn": cfg.Tnn, "levels": len(levels), "windows_per_frame": windows_per_frame,
                       "parallelism": f"frame-sharded dp{world}",
                       "dist_backend": backend, "ranks_per_gpu": (world + n_dev - 1) // n_dev if world > 1 else 1,
                       "l2": "inputs larger than L2 (%.0f MB frames/step/GPU)" % (frames.nbytes / 1e6)},
            "stage1_gwindows_per_s": windows_per_frame * batch / (s1_avg_ms / 1000.0) / 1e9 * world,
            "pipeline_gwindows_per_s": windows_per_frame * total_frames / (ms / 1000.0) / 1e9,
            "stage_ms_per_step": {k: v for k, v in zip(["h2d", "pyramid", "stage1", "selective", "nms_out"],
                                                        stats["ms"])},
            "stage_ms_alone": {k: v for k, v in zip(["h2d", "pyramid", "stage1", "selective", "nms_out"], alone)},
            # pyramid: frame read once + levels written once (algorithmic bytes) / its time alone
            "pyramid_gbs_alone": (frames.nbytes + batch * sum(((w + 15) // 16 * 16) * h for _, w, h in levels))
                                 / (alone[1] / 1000.0) / 1e9 if alone[1] > 0 else None,
            "table1_counts_last_step": {k: stats[k] for k in ("windows", "stage1", "stage2", "stage3", "nms")},
            "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": tc_peak,
                         "unit": "TFLOP/s", "frac": achieved_tflops / tc_peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes": int(batch * sum(((w + 15) // 16 * 16) * h for _, w, h in levels)),
                         "kernel": "stage1_tc_kernel",
                         "peak_note": "dense fp16/bf16 tensor peak, measured burst "
                                      "(MEASURED_PEAKS.json bf16_tflops; the ~15 ms timed region runs at "
                                      "the max SM clock); achieved = ALGORITHMIC fp32-equivalent FLOPs of "
                                      "CNN1 / measured stage-1 time. The MMAs actually issued "
                                      "(mma_issued_*) are several times that (hi+lo splits, implicit-GEMM "
                                      "zero taps; DESIGN.md K2)",
                         "fp32_ffma_peak": fp32_peak,
                         "frac_of_fp32_ffma_peak": achieved_tflops / fp32_peak,
                         # fp32 accuracy costs 2 (layer 1) or 3 (layers 2-3) fp16 MMAs per
                         # product: the fp16 peak divided by that FLOP-weighted factor is the
                         # most fp32-accurate work the tensor cores can do (K2)
                         "fp32_split_mmas_per_product": split_mma_factor(levels),
                         "fp32_split_peak": tc_peak / split_mma_factor(levels),
                         "frac_of_fp32_split_peak": achieved_tflops * split_mma_factor(levels) / tc_peak,
                         # the tensor work the kernel actually issues (all MMAs, zero taps and
                         # hi/lo splits included) over the same time: how busy the tensor
                         # cores are, as opposed to how much of it the algorithm needs
                         "mma_issued_tflops": mma_flops / (s1_ms / 1000.0) / 1e12 if s1_ms > 0 else None,
                         "mma_issued_frac": mma_flops / (s1_ms / 1000.0) / 1e12 / tc_peak if s1_ms > 0 else None},
            "e2e": {"value": world * batch * e2e_steps / (ms_e2e / 1000.0), "unit": "frames/s",
                    "h2d_bytes_per_step": int(frames.nbytes), "d2h_bytes_per_step": int(d2h // e2e_steps),
                    "h2d_gbs_achieved": int(frames.nbytes) * e2e_steps / (ms_e2e / 1000.0) / 1e9,
                    "h2d_gbs_copy_alone": h2d_gbs, "host_numa": numa},
            "latency_batch1_ms": {"wall_median": float(np.median(lat_wall)),
                                  "wall_p90": float(np.percentile(lat_wall, 90)),
                                  "device_median": float(np.median(lat_dev)),
                                  "call": "synchronous ccnn_detect of 1 device-resident frame"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if merge_check is not None:
            line["merge_check"] = merge_check
        # SURVEY §8(d) / the bench contract: the oracle baseline on rank 0 at N=1 only
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, ws, frames, T1, T2)
        print(json.dumps(line), flush=True)
    det.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

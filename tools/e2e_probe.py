"""Where the end-to-end (pinned host frames) path loses to the plain H2D copy: the copy alone
(1-D and as the 2-D copy the runtime issues), a synchronous detect's H2D event time, and the
streamed loop's per-batch H2D times.  usage: python tools/e2e_probe.py [c4] [batches]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from cuda.bindings import runtime as cudart
from paper_1508_01292_b200 import Detector
from synth import arch, configs, weights

cfg = configs.BY_ID[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
frames = cfg.make_frames(cfg.batch)
host = torch.from_numpy(frames).pin_memory()
dev = torch.empty_like(host, device="cuda")
nb = host.numel()
s = torch.cuda.current_stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ms1 = timed(lambda: dev.copy_(host, non_blocking=True))
W, H = cfg.width, cfg.height
rows = H * cfg.batch
ms2 = timed(lambda: cudart.cudaMemcpy2DAsync(dev.data_ptr(), W, host.data_ptr(), W, W, rows,
                                             cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream))
print(f"copy alone 1-D: {nb / ms1 / 1e6:.1f} GB/s   2-D ({rows} rows of {W} B): {nb / ms2 / 1e6:.1f} GB/s")

ws = weights.make_cascade_weights()
T1, T2 = cfg.thresholds()
det = Detector(arch.NETS, ws, T1, T2, cfg.Tnn, cfg.rule, max_w=cfg.width, max_h=cfg.height,
               max_batch=cfg.batch, queue_capacity=max(4096, 40000 if cfg.kind == "clutter" else 0))
for _ in range(3):
    det.detect(host, cfg.min_face, cfg.scale_step)
print("synchronous detect of host frames: h2d %.3f ms (%.1f GB/s), stages %s" % (
    det.last_stats["ms"][0], nb / det.last_stats["ms"][0] / 1e6,
    [round(float(x), 3) for x in det.last_stats["ms"]]))
opts = sys.argv[3:]
if "setstream" in opts:
    det.set_stream(torch.cuda.current_stream().cuda_stream)
if "clocks" in opts:
    import bench
    cs = bench.ClockSampler(0)
    cs.start()
if "devfirst" in opts:                  # bench.py's order: a device-frame streamed loop first
    dfr = host.cuda()
    for _ in range(2):
        det.submit(dfr, cfg.min_face, cfg.scale_step)
    for k in range(20):
        if k + 2 < 20:
            det.submit(dfr, cfg.min_face, cfg.scale_step)
        det.collect()
    for _ in range(3):
        det.detect(dfr, cfg.min_face, cfg.scale_step)
    det.detect(host, cfg.min_face, cfg.scale_step)
torch.cuda.synchronize()
t0 = time.perf_counter()
h2d = []
tm = "untimed" not in opts
if "bind" in opts:
    import bench
    print(bench.bind_host_to_gpu(0)[1])
for _ in range(2):
    det.submit(host, cfg.min_face, cfg.scale_step, timed=tm)
for k in range(n):
    if k + 2 < n:
        det.submit(host, cfg.min_face, cfg.scale_step, timed=tm)
    det.collect()
    h2d.append(det.last_stats["ms"][0])
dt = time.perf_counter() - t0
print(opts, "streamed: %.1f frames/s, %.1f GB/s of frames; per-batch h2d event ms %s" % (
    n * cfg.batch / dt, n * nb / dt / 1e9, [round(x, 2) for x in h2d]))

"""Host-side cost of ccnn_submit / ccnn_collect per batch (streamed, device frames) vs the
device step: is a small-frame config host-bound?  usage: python tools/host_overhead.py [c1] [n]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1508_01292_b200 import Detector
from synth import arch, configs, weights

cfg = configs.BY_ID[sys.argv[1] if len(sys.argv) > 1 else "c1"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ws = weights.make_cascade_weights()
T1, T2 = cfg.thresholds()
det = Detector(arch.NETS, ws, T1, T2, cfg.Tnn, cfg.rule, max_w=cfg.width, max_h=cfg.height,
               max_batch=cfg.batch, queue_capacity=max(4096, 40000 if cfg.kind == "clutter" else 0))
fr = torch.from_numpy(cfg.make_frames(cfg.batch)).cuda()
for _ in range(2):
    det.submit(fr, cfg.min_face, cfg.scale_step)
ts, tc = [], []
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    a = time.perf_counter()
    det.submit(fr, cfg.min_face, cfg.scale_step)
    b = time.perf_counter()
    det.collect()
    c = time.perf_counter()
    ts.append(b - a)
    tc.append(c - b)
t1 = time.perf_counter()
for _ in range(2):
    det.collect()
print(cfg.name, "per batch: wall %.1f us, submit %.1f us (median), collect %.1f us (median, includes the wait)"
      % ((t1 - t0) / n * 1e6, np.median(ts) * 1e6, np.median(tc) * 1e6))

"""Content dependence of the frame time (the analogue of PAPER.md Fig. 11, P:243 / P:131:
"nearly constant processing time ... even when there is a significant increase in the number
of faces"): C4 4K frames (min face 60, scale 1.2, 32 frames per step, three batches in flight
as in bench.py), T1 moved so that the stage-1 survival rate sweeps 5e-5 .. 1e-2 (T2 as
calibrated for C4).  Thresholds come from quantiles of the GPU's own dense stage-1 map of two
frames (a performance sweep: no parity claim).  One JSON line per rate.

usage (GPU box): python tools/survival_sweep.py [out.jsonl] [steps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1508_01292_b200 import Detector, ccnn  # noqa: E402
from synth import arch, configs, weights  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/survival_sweep.jsonl"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = configs.C4
ws = weights.make_cascade_weights()
T1c, T2 = c.thresholds()
fr = torch.from_numpy(c.make_frames()).cuda()
# score distribution: dense stage-1 maps of two frames
probe = Detector(arch.NETS, ws, T1c, T2, c.Tnn, c.rule, max_w=c.width, max_h=c.height, max_batch=2)
probe.set_debug(ccnn.CCNN_DEBUG_STAGE1)
probe.detect(fr[:2], c.min_face, c.scale_step)
scores = np.concatenate([probe.stage1_map(f, l).ravel() for f in range(2)
                         for l in range(len(probe.levels(f)))])
probe.close()
rows = []
for rate in (5e-5, 1e-4, 3e-4, 1e-3, 3e-3, 1e-2):
    T1 = float(np.float32(np.quantile(scores, 1.0 - rate)))
    det = Detector(arch.NETS, ws, T1, T2, c.Tnn, c.rule, max_w=c.width, max_h=c.height,
                   max_batch=c.batch, queue_capacity=max(4096, int(4 * rate * 316848)))
    for _ in range(3):
        det.detect(fr, c.min_face, c.scale_step)
    st = det.last_stats
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stage = np.zeros(5)
    det.submit(fr, c.min_face, c.scale_step)
    det.submit(fr, c.min_face, c.scale_step)
    for k in range(steps):
        if k + 2 < steps:
            det.submit(fr, c.min_face, c.scale_step)
        det.collect()
        stage += np.array(det.last_stats["ms"])
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    alone = []
    for _ in range(3):
        det.detect(fr, c.min_face, c.scale_step)
        alone.append(det.last_stats["ms"])
    row = {"target_rate": rate, "T1": T1, "survival_rate": st["stage1"] / st["windows"],
           "survivors_per_frame": st["stage1"] / c.batch, "stage2_per_frame": st["stage2"] / c.batch,
           "accepted_per_frame": st["stage3"] / c.batch, "boxes_per_frame": st["nms"] / c.batch,
           "ms_per_step": ms, "us_per_frame": 1000.0 * ms / c.batch,
           "frames_per_s": c.batch / (ms / 1000.0),
           "stage_ms_per_step": dict(zip(["h2d", "pyramid", "stage1", "selective", "nms_out"],
                                         (stage / steps).round(4).tolist())),
           "stage_ms_alone": dict(zip(["h2d", "pyramid", "stage1", "selective", "nms_out"],
                                      np.median(np.array(alone), axis=0).round(4).tolist()))}
    rows.append(row)
    print(json.dumps(row), flush=True)
    det.close()
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
with open(out_path, "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")

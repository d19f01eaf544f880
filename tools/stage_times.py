"""Per-stage device times of synchronous ccnn_detect calls (no batch overlap): median over
--reps calls of one config.  usage: [CCNN_LIB_VARIANT=v] python tools/stage_times.py [c4] [reps]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1508_01292_b200 import Detector
from synth import arch, configs, weights

cfg = configs.BY_ID[sys.argv[1] if len(sys.argv) > 1 else "c4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ws = weights.make_cascade_weights()
T1, T2 = cfg.thresholds()
det = Detector(arch.NETS, ws, T1, T2, cfg.Tnn, cfg.rule, max_w=cfg.width, max_h=cfg.height,
               max_batch=cfg.batch, queue_capacity=max(4096, 40000 if cfg.kind == "clutter" else 0))
fr = torch.from_numpy(cfg.make_frames(cfg.batch)).cuda()
ms = []
for k in range(reps + 3):
    det.detect(fr, cfg.min_face, cfg.scale_step)
    if k >= 3:
        ms.append(det.last_stats["ms"])
ms = np.median(np.array(ms), axis=0)
print(os.environ.get("CCNN_LIB_VARIANT", "default"), cfg.name,
      dict(zip(["h2d", "pyramid", "stage1", "selective", "nms_out"], [round(float(x), 4) for x in ms])))

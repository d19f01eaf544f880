"""Run the C4 batch once with libccnn_prof.so (built with -DS1_PROFILE) and print the
per-role stage-1 barrier-wait vs busy cycle totals (units of 64 cycles, summed over warps)."""
import os, sys
os.environ["CCNN_LIB_VARIANT"] = sys.argv[1] if len(sys.argv) > 1 else "prof"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1508_01292_b200 import Detector
from synth import arch, configs, weights
c = configs.C4
T1, T2 = c.thresholds()
fr = torch.from_numpy(c.make_frames()).cuda()
det = Detector(arch.NETS, weights.make_cascade_weights(), T1, T2, c.Tnn, c.rule, max_batch=32)
for _ in range(3):
    det.detect(fr, c.min_face, c.scale_step)
k = det.counters()
print({"L1_wait": k[0], "L23_wait": k[1], "L1_busy": k[2], "L23_busy": k[3],
       "L1_wait_frac": k[0] / max(1, k[0] + k[2]), "L23_wait_frac": k[1] / max(1, k[1] + k[3]),
       "stage1_ms": det.last_stats["ms"][2]})

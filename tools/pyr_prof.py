"""Run a config's batch through both pyramid forms (tld4 texture gathers via
CCNN_DEBUG_PYR_TEX, then byte gathers) and print the pyramid event times; for ncu captures
of both kernels.  usage: python tools/pyr_prof.py [C1..C5]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1508_01292_b200 import Detector, ccnn
from synth import arch, configs, weights
c = getattr(configs, sys.argv[1] if len(sys.argv) > 1 else "C4")
T1, T2 = c.thresholds()
fr = torch.from_numpy(c.make_frames()).cuda()
det = Detector(arch.NETS, weights.make_cascade_weights(), T1, T2, c.Tnn, c.rule,
               max_batch=max(32, fr.shape[0]))
for flag, name in ((ccnn.CCNN_DEBUG_PYR_TEX, "tex"), (0, "ldg")):
    det.set_debug(flag)
    ms = []
    for _ in range(6):
        det.detect(fr, c.min_face, c.scale_step)
        ms.append(det.last_stats["ms"][1])
    print(name, "pyramid ms", sorted(ms[1:])[len(ms[1:]) // 2])

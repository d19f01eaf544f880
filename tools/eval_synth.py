"""NEXT #3 evaluation run: the detector (libccnn.so, ccnn_detect_frames) on variable-size
synthetic stills with planted faces, scored with the paper's two protocols
(paper_1508_01292_b200/evaluate.py):

* "fddb": 64 stills of mixed sizes <= 0.25 MP (as FDDB), minSize 15, scaleFactor
  1.05, T_nn 1; discrete ROC over the box-score threshold + continuous score;
* "afw": 12 stills of 0.5-5 MP (as AFW), minSize 80, scaleFactor 1.1;
  precision / recall / F1 with the 44-variant test, mean F1 over T_nn = {1, 2, 3}.

The cascade weights are the seeded random initialisation (trained weights are out of scope),
so the numbers characterise the harness and the planted-face workload, not a trained
detector.  usage: python tools/eval_synth.py [--out FILE]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_01292_b200 import Detector, evaluate as ev   # noqa: E402
from synth import arch, configs, frames as synth_frames, weights   # noqa: E402


def stills(n, lo_px, hi_px, min_face, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        while True:
            w, h = int(rng.integers(lo_px[0], hi_px[0] + 1)), int(rng.integers(lo_px[1], hi_px[1] + 1))
            if w * h <= hi_px[0] * hi_px[1]:
                break
        img, gt = synth_frames.make_still_gt(w, h, seed + 17 * k, min_face,
                                             n_faces=int(rng.integers(1, 6)))
        out.append((img, gt))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    T1, T2 = configs.C4.thresholds()
    ws = weights.make_cascade_weights()
    res = {"weights": "seeded random init (no trained weights: out of scope)", "T1": T1, "T2": T2}

    # ---- FDDB-like ----
    data = stills(64, (250, 250), (500, 500), 15, 4242)
    det = Detector(arch.NETS, ws, T1, T2, 1, 0, max_w=512, max_h=512, max_batch=64,
                   queue_capacity=16384)
    t0 = time.time()
    boxes = det.detect_frames([d[0] for d in data], 15, 1.05)
    t_fddb = time.time() - t0
    per = ev.boxes_by_frame(boxes, len(data))
    scores = np.concatenate([p[1] for p in per]) if len(boxes) else np.zeros(0)
    ths = sorted(set([-2.0] + [float(q) for q in np.quantile(scores, np.linspace(0, 1, 11))])) \
        if len(scores) else [-2.0]
    roc = ev.score_fddb([(d[1], p[0], p[1]) for d, p in zip(data, per)], ths)
    res["fddb"] = dict(images=len(data), faces=sum(len(d[1]) for d in data),
                       sizes=[list(d[0].shape[::-1]) for d in data[:8]] + ["..."],
                       min_face=15, scale_step=1.05, Tnn=1, boxes=int(len(boxes)),
                       stats=det.last_stats, wall_s=t_fddb, roc=roc)
    det.close()

    # ---- AFW-like ----
    data = stills(12, (900, 600), (2500, 2000), 80, 777)
    f1s, runs = [], []
    for tnn in (1, 2, 3):
        d3 = Detector(arch.NETS, ws, T1, T2, tnn, 0, max_w=2560, max_h=2048, max_batch=16,
                      queue_capacity=16384)
        b = d3.detect_frames([d[0] for d in data], 80, 1.1)
        per = ev.boxes_by_frame(b, len(data))
        r = ev.score_afw([(d[1], p[0]) for d, p in zip(data, per)])
        r["Tnn"] = tnn
        r["boxes"] = int(len(b))
        runs.append(r)
        f1s.append(r["f1"])
        d3.close()
    res["afw"] = dict(images=len(data), faces=sum(len(d[1]) for d in data), min_face=80,
                      scale_step=1.1, runs=runs, mean_f1=float(np.mean(f1s)))
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

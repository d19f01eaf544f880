"""Steady-state timeline of the streamed path (three batches in flight, device frames):
CCNN_TIMELINE=1 makes ccnn_collect print each batch's event times (ms since the first
pyramid); this summarises them per batch: pyramid duration, stage-1 duration, tail, and the
spacing of consecutive stage-1 starts (= the step).
usage: python tools/timeline.py [c4] [batches] [host]   (host: pinned host frames, H2D inside)"""
import os, re, subprocess, sys

if os.environ.get("CCNN_TIMELINE") != "1":
    env = dict(os.environ, CCNN_TIMELINE="1")
    r = subprocess.run([sys.executable] + sys.argv, env=env, capture_output=True, text=True)
    sys.stdout.write(r.stdout)
    f = r"(-?[\d.]+)"
    pat = re.compile(r"batch (\d+): pyr %s-%s s1 %s-%s sel-%s end %s h2d %s-%s" % ((f,) * 8))
    rows = [tuple(float(x) for x in m.groups()) for m in pat.finditer(r.stderr)]
    if not rows:
        sys.stderr.write(r.stderr[-3000:])
        sys.exit(1)
    print("batch  pyr_ms  s1_ms  sel+nms_ms  s1_start_gap  s1_wait_after_pyr  h2d_ms  h2d_gap_ms")
    prev = None
    prev_h = None
    for b, p0, p1, s0, s1, se, e, h0, h1 in rows:
        gap = s0 - prev if prev is not None else float("nan")
        hg = h0 - prev_h if prev_h is not None else float("nan")
        print(f"{int(b):5d}  {p1 - p0:6.3f}  {s1 - s0:5.3f}  {e - s1:10.3f}  {gap:12.3f}  {s0 - p1:17.3f}"
              f"  {h1 - h0:6.3f}  {hg:10.3f}")
        prev = s0
        prev_h = h1
    rows = [r[:7] for r in rows]
    tail = rows[len(rows) // 2:]
    import statistics as st
    print("median (second half): pyr %.3f  s1 %.3f  tail %.3f  step %.3f" % (
        st.median(r[2] - r[1] for r in tail), st.median(r[4] - r[3] for r in tail),
        st.median(r[6] - r[4] for r in tail),
        st.median(tail[i][3] - tail[i - 1][3] for i in range(1, len(tail)))))
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1508_01292_b200 import Detector
from synth import arch, configs, weights

cfg = configs.BY_ID[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ws = weights.make_cascade_weights()
T1, T2 = cfg.thresholds()
det = Detector(arch.NETS, ws, T1, T2, cfg.Tnn, cfg.rule, max_w=cfg.width, max_h=cfg.height,
               max_batch=cfg.batch, queue_capacity=max(4096, 40000 if cfg.kind == "clutter" else 0))
fr = torch.from_numpy(cfg.make_frames(cfg.batch))
fr = fr.pin_memory() if "host" in sys.argv[3:] else fr.cuda()
for _ in range(2):
    det.submit(fr, cfg.min_face, cfg.scale_step)
for _ in range(n):
    det.submit(fr, cfg.min_face, cfg.scale_step)
    det.collect()
for _ in range(2):
    det.collect()

"""Markdown results table of the bench lines in profiles/ (DESIGN.md §6).
usage: python tools/results_table.py [tag]   (tag: r2 -> profiles/r2_bench_c*.json)"""
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
names = {"c1": "C1 320×240, min 24", "c2": "C2 256 stills 450×450, min 15", "c3": "C3 1080p, min 40",
         "c4": "**C4 4K, min 60 (headline)**", "c5": "C5 4K clutter (1% survival)"}
print("| config | frames / step | frames/s | ms / step | stage 1 ms | Gwindows/s (stage 1) | "
      "e2e frames/s (host frames) | roofline frac (mma issued) |")
print("|---|---|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4", "c5"):
    p = os.path.join(root, f"{tag}_bench_{c}.json")
    if not os.path.exists(p):
        continue
    d = json.loads(open(p).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"| {names[c]} | {d['config']['frames_per_step_per_gpu']} | {d['value']:,.0f} | "
          f"{d['ms_per_step']:.3f} | {d['stage_ms_per_step']['stage1']:.3f} | "
          f"{d['stage1_gwindows_per_s']:.1f} | {d['e2e']['value']:,.0f} | "
          f"{r['frac']:.3f} ({r.get('mma_issued_frac', float('nan')):.2f}) |")

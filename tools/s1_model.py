"""Model of the stage-1 kernel's executed FFMA vs algorithmic MACs for band width TW,
CTA column count NT (=2TW+10) and segment height (DESIGN.md "Stage 1" design study)."""
import math, sys
sys.path.insert(0, '.')
from bench import level_table

def alg_macs(levels):
    t = 0
    for _, lw, lh in levels:
        nx, ny = (lw - 27)//4 + 1, (lh - 31)//4 + 1
        t += (4*nx+20)*(4*ny+24)*96 + (2*nx+8)*(2*ny+10)*324 + nx*ny*362
    return t

def executed(levels, TW, seg, l3win=1):
    NT = 2*TW + 10
    P2 = TW + 4
    ffma = steps = 0
    for _, lw, lh in levels:
        nx, ny = (lw - 27)//4 + 1, (lh - 31)//4 + 1
        nseg = max(1, math.ceil(ny/seg)); rows = math.ceil(ny/nseg)
        for x0 in range(0, nx, TW):
            for y0 in range(0, ny, rows):
                nr = min(rows, ny - y0)
                ffma += NT*768*(nr+6) + P2*1296*(nr+5) + TW*362*(nr+5)
                steps += nr + 8
    return ffma, steps

for name, (W, H, mf, sf) in {"c4": (3840, 2160, 60, 1.2), "c3": (1920, 1080, 40, 1.2), "c1": (320, 240, 24, 1.2), "c2": (450,450,15,1.05)}.items():
    lv = level_table(W, H, mf, sf)
    a = alg_macs(lv)
    for TW in (27, 59, 123):
        for seg in (32, 64, 128, 10**6):
            e, st = executed(lv, TW, seg)
            print(f"{name} TW={TW:3d} seg={seg:7d}: useful/executed FFMA = {a/e:.3f}  steps/frame={st}")

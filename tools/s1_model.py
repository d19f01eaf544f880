"""Executed-vs-algorithmic FFMA model of the stage-1 kernel (v5+, patchwork bands):
TW = 59 windows per band, 2 window rows per super-step, L1/L2 computed for all 128/64
columns of a band; tails packed first-fit by height (runtime.cu build_plan)."""
import math, sys
sys.path.insert(0, '.')
from bench import level_table

TW, GAP, MAXP = 59, 6, 4

def alg_macs(levels):
    t = 0
    for _, lw, lh in levels:
        nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
        t += (4*nx+20)*(4*ny+24)*96 + (2*nx+8)*(2*ny+10)*324 + nx*ny*362
    return t

def bands(levels):
    out, tails = [], []
    for _, lw, lh in levels:
        nx, ny = (lw - 27) // 4 + 1, (lh - 31) // 4 + 1
        out += [ny] * (nx // TW)
        if nx % TW: tails.append((ny, nx % TW))
    tails.sort(reverse=True)
    tb = []
    for ny, w in tails:
        for b in tb:
            if b[2] < MAXP and b[1] + GAP + w <= TW:
                b[1] += GAP + w; b[2] += 1; break
        else:
            tb.append([ny, w, 1])
    return out + [b[0] for b in tb]

def executed(levels, seg):
    ffma = 0
    for h in bands(levels):
        nseg = max(1, math.ceil(h / seg)); rows = math.ceil(h / nseg)
        for y0 in range(0, h, rows):
            nr = min(rows, h - y0)
            steps = (nr + 7) // 2 + 1                 # super-steps (2 window rows each)
            ffma += steps * 128 * (2 * 768 + 1296 + 360)   # per thread per super-step
    return ffma

if __name__ == "__main__":
    for name, (W, H, mf, sf) in {"c4": (3840, 2160, 60, 1.2), "c3": (1920, 1080, 40, 1.2),
                                 "c1": (320, 240, 24, 1.2), "c2": (450, 450, 15, 1.05)}.items():
        lv = level_table(W, H, mf, sf)
        a = alg_macs(lv)
        print(name, " ".join(f"seg{seg}={a / executed(lv, seg):.3f}" for seg in (32, 64, 128, 256, 10**5)))

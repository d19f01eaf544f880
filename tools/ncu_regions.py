"""Per-region stall attribution from an ncu source page (SASS).  usage:
python tools/ncu_regions.py src.csv  -- regions = backward-branch loops, printed with stalls."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
base = int(data[0][col["Address"]], 16)
ins = [(int(r[col["Address"]], 16) - base, r[col["Source"]].strip(), r) for r in data]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
loops = []
for i, (a, t, _) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+.*?0x([0-9a-f]+)", t)
    if m:
        ta = int(m.group(1), 16) - base
        if ta < a:
            loops.append((ta, a))
loops.sort(key=lambda x: x[1] - x[0])
def region(a):
    for lo, hi in loops:
        if lo <= a <= hi: return f"{lo:#x}-{hi:#x}"
    return "outside"
agg = collections.defaultdict(lambda: collections.Counter())
execd = collections.Counter(); ninst = collections.Counter()
for a, t, r in ins:
    g = region(a)
    for h in reasons:
        v = r[col[h]]
        if v and v != "0": agg[g][h] += int(float(v))
    execd[g] += int(float(r[col["Instructions Executed"]] or 0)); ninst[g] += 1
tot = sum(sum(c.values()) for c in agg.values())
for g in sorted(agg, key=lambda g: -sum(agg[g].values())):
    c = agg[g]; s = sum(c.values())
    print(f"{g:16s} static={ninst[g]:5d} exec={execd[g]:.3e} samples={s/tot:6.1%}  " +
          " ".join(f"{k[6:]}={v/s:.0%}" for k, v in c.most_common(6)))

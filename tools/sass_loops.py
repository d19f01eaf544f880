"""Instruction mix per loop (backward-branch region) of build_tools/mix.sass (tools/sass_mix.sh)."""
import re, collections
ins = []
for l in open('build_tools/mix.sass'):
    m = re.match(r'\s+/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for a, t in ins:
    m = re.search(r'BRA(?:\.U)?\s+(?:U?P\d+,\s*)?0x([0-9a-f]+)', t)
    if m and int(m.group(1), 16) < a: loops.append((int(m.group(1), 16), a))
for lo, hi in sorted(loops, key=lambda x: x[1] - x[0]):
    body = [t for a, t in ins if lo <= a <= hi]
    c = collections.Counter(t.split()[0] if not t.startswith('@') else t.split()[1] for t in body)
    print(f"{lo:#x}-{hi:#x} n={len(body)} FFMA={c['FFMA']} ", c.most_common(12))

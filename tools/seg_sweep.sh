#!/bin/bash
# stage-1 ms per 32-frame 4K batch for several segment heights
for seg in 0 32 64 128 256 16384; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 --seg $seg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('seg', $seg, 'stage1_ms', round(d['stage_ms_per_step']['stage1'],4), 'frac', round(d['roofline']['frac'],4), 'fps', round(d['value']))"
done

#!/bin/bash
# usage: tools/variant_bench.sh v1 v2 ...  -- stage timings of each in-tree libccnn_<v>.so ("" = default)
for v in "$@"; do
  [ "$v" = "default" ] && v=""
  CCNN_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-default}', round(d['value']), d['stage_ms_per_step'], d['roofline']['frac'])"
done

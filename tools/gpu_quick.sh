#!/bin/bash
# quick GPU check: parity tests (first failure stops), then a short bench.  usage: tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
K=${2:-}
if [ -n "$K" ]; then KA=(-k "$K"); else KA=(); fi
timeout 600 python -m pytest tests -m gpu -q -x "${KA[@]}" 2>&1 | tail -25 > gpurun_out/tests_$TAG.log
cat gpurun_out/tests_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json

#!/bin/bash
# one GPU round trip: parity tests, bench, stage-1 ncu capture.  usage: tools/gpu_cycle.sh TAG
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/tests_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage1 -s 3 -c 1 -o gpurun_out/prof_s1_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
cat gpurun_out/tests_$TAG.log; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json

#!/bin/bash
# one GPU round trip: parity tests, bench, launch list, stage-1 ncu capture.  usage: tools/gpu_cycle.sh TAG [noprof]
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/tests_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
if [ "$2" != "noprof" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage1 -s 3 -c 1 -o gpurun_out/prof_s1_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
fi
cat gpurun_out/tests_$TAG.log; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/launches_$TAG.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    print("launch", r[ki][:60], r[vi])
PY

#!/bin/bash
# Round-end evidence on one B200: tests, benches of every config, launch list, ncu captures,
# compute-sanitizer.  Everything lands in gpurun_out/; summaries are copied to profiles/.
set -x
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -20 > gpurun_out/tests_$TAG.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
for c in c1 c2 c3 c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 8 --csv --log-file gpurun_out/launches_c4_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for k in stage1 pyramid selective nms; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${k}_$TAG.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:selective -s 2 -c 1 -o gpurun_out/prof_selective_c5_$TAG python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_selective_c5_$TAG.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -k "c1_parity_calibrated or edge_cases or rgb_ingest or mixed_size_frames_api" > gpurun_out/memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_$TAG.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -k "c1_parity_calibrated or segment_heights_and_patchwork and 3" > gpurun_out/racecheck_$TAG.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_$TAG.log
tail -3 gpurun_out/tests_$TAG.log; tail -n 2 gpurun_out/memcheck_$TAG.log; tail -n 2 gpurun_out/racecheck_$TAG.log

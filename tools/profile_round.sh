#!/bin/bash
# Round-end evidence on one B200: tests, benches of every config, launch list, ncu captures,
# compute-sanitizer, the survival sweep.  Everything lands in gpurun_out/; summaries are copied
# to profiles/ by hand.   usage: bash tools/profile_round.sh TAG [parts...]
# parts: tests bench launches ncu sanitize sweep (default: all)
set -x
TAG=${1:-r2}; shift
PARTS=${@:-tests bench launches ncu sanitize sweep}
mkdir -p gpurun_out
has() { [[ " $PARTS " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/tests_$TAG.log 2>&1
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
fi
if has bench; then
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
  for c in c1 c2 c3 c5; do
    timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-traffic > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  done
  timeout 400 python bench.py --gpus 2 --dist-backend gloo --steps 10 --no-cpu-baseline --no-traffic > gpurun_out/bench_g2gloo_$TAG.json 2> gpurun_out/bench_g2gloo_$TAG.err
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1
fi
if has launches; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 12 --csv --log-file gpurun_out/launches_c4_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-traffic --e2e-steps 1 > /dev/null 2>&1
fi
if has ncu; then
  for k in ${NCU_KERNELS:-stage1_tc pyramid_gather4 selective_cnn2 selective_kernel nms}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_$TAG python tools/stage_times.py c4 2 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  done
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:selective_cnn2 -s 1 -c 1 -o gpurun_out/prof_cnn2_c5_$TAG python tools/stage_times.py c5 1 > gpurun_out/ncu_cnn2_c5_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"selective_kernel|nms" -s 2 -c 2 -o gpurun_out/prof_cnn3nms_c5_$TAG python tools/stage_times.py c5 1 > gpurun_out/ncu_cnn3nms_c5_$TAG.log 2>&1
fi
if has sanitize; then
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nms.py tests/test_gpu_stress.py -q -k "c1_parity_calibrated or edge_cases or rgb_ingest or mixed_size_frames_api or clutter or chains or capacity or streamed or streaming_submit" > gpurun_out/memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_$TAG.log
  timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nms.py -q -k "c1_parity_calibrated or segment_heights_and_patchwork and 3 or clutter_sets and 4096 or chains" > gpurun_out/racecheck_$TAG.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_$TAG.log
  timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nms.py tests/test_gpu_stress.py -q -k "c1_parity_calibrated or clutter_sets and 4096 or chains or streamed" > gpurun_out/synccheck_$TAG.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck_$TAG.log
fi
if has sweep; then
  timeout 600 python tools/survival_sweep.py gpurun_out/survival_sweep_$TAG.jsonl 20 > gpurun_out/survival_sweep_$TAG.log 2>&1
fi
tail -3 gpurun_out/tests_$TAG.log 2>/dev/null; tail -n 2 gpurun_out/memcheck_$TAG.log gpurun_out/racecheck_$TAG.log gpurun_out/synccheck_$TAG.log 2>/dev/null; cat gpurun_out/survival_sweep_$TAG.jsonl 2>/dev/null | cut -c1-200

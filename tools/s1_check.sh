# stage-1 change check: parity subset, stage times (c4 c3 c2 c5), pipelined C4 bench
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_parity_low or ragged_multi_frame_batch or edge or fddb_like or mixed_size_frames_parity or segment_heights or c4_debug_map or host_vs or streaming_device" 2>&1 | tail -2
for c in c4 c3 c2 c5; do timeout 120 python tools/stage_times.py $c 5; done
timeout 300 python bench.py --no-cpu-baseline --no-traffic --steps 40 > gpurun_out/bench_s1chk.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_s1chk.json')); print('bench', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms_per_step'].items()}, d['roofline']['frac'])"

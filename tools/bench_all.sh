# quick pipelined bench of every config (no cpu baseline / traffic): value, ms/step, stage times
for c in "$@"; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-traffic --steps 20 > gpurun_out/bench_q_$c.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_q_$c.json')); print('$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms_per_step'].items()}, 'lat1', round(d['latency_batch1_ms']['wall_median'],4))"; done

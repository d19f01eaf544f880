# selective grid sizes vs the pipelined step (C4 / C5), experiment knobs CCNN_SEL_GRID / CCNN_CNN3_SMS
for c in c4 c5; do for g in 0 96 64 32; do for g3 in 0 32; do
  CCNN_SEL_GRID=$g CCNN_CNN3_SMS=$g3 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-traffic 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'sel', $g, 'cnn3', $g3, round(d['value']), round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})"
done; done; done

for seg in 0 160 120; do
 timeout 300 python bench.py --config c4 --seg $seg --no-cpu-baseline --no-traffic --steps 30 > gpurun_out/bg.json 2>/dev/null
 python -c "import json; d=json.load(open('gpurun_out/bg.json')); print('seg $seg', round(d['value']), round(d['ms_per_step'],4), round(d['stage_ms_per_step']['stage1'],4))"
done
for g in 0 128 100; do
 CCNN_SEL_GRID=$g timeout 300 python bench.py --config c4 --no-cpu-baseline --no-traffic --steps 30 > gpurun_out/bg.json 2>/dev/null
 python -c "import json; d=json.load(open('gpurun_out/bg.json')); print('selgrid $g', round(d['value']), round(d['ms_per_step'],4))"
done
for g in 0 100 64; do
 CCNN_CNN3_SMS=$g timeout 300 python bench.py --config c4 --no-cpu-baseline --no-traffic --steps 30 > gpurun_out/bg.json 2>/dev/null
 python -c "import json; d=json.load(open('gpurun_out/bg.json')); print('cnn3sms $g', round(d['value']), round(d['ms_per_step'],4))"
done

# A/B of library variants (built in-tree as libccnn_<name>.so): C4 stage times + pipelined bench
# usage: bash tools/variant_bench.sh default name1 name2 ...
for v in "$@"; do if [ $v = default ]; then unset CCNN_LIB_VARIANT; else export CCNN_LIB_VARIANT=$v; fi
timeout 120 python tools/stage_times.py c4 5
timeout 300 python bench.py --no-cpu-baseline --no-traffic --steps 40 > gpurun_out/bench_v_$v.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_v_$v.json')); print('$v', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms_per_step'].items()})"; done

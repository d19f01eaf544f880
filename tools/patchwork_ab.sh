# patchwork (tail pieces packed into shared bands) on / off: stage-1 time alone and the
# pipelined bench, C1-C4; plus parity with patchwork off
CCNN_PATCHWORK=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_parity_low or ragged_multi_frame_batch and ldg or segment_heights or fddb_like" 2>&1 | tail -1
for c in c1 c2 c3 c4; do for pw in 1 0; do
  CCNN_PATCHWORK=$pw timeout 120 python tools/stage_times.py $c 5 | sed "s/^/pw=$pw /"
  CCNN_PATCHWORK=$pw timeout 300 python bench.py --config $c --no-cpu-baseline --no-traffic --steps 20 > gpurun_out/b_pw.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/b_pw.json')); print('pw=$pw $c bench', round(d['value']), round(d['ms_per_step'],4))"
done; done

#!/bin/bash
# Pyramid experiments on one B200: stage times of library variants built with different
# pyramid class thresholds, plus ncu captures of the pyramid kernels (C4).
# usage (on the GPU box): bash tools/pyr_variants.sh TAG "variant:DEFINE ..." ...
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python paper_1508_01292_b200/build.py $name $defs > /dev/null 2>&1 || echo "build $name failed"
done
for spec in "$@"; do
  name=${spec%%:*}
  CCNN_LIB_VARIANT=$name timeout 120 python tools/stage_times.py c4 10 >> gpurun_out/pyr_${TAG}.txt 2>&1
  CCNN_LIB_VARIANT=$name timeout 120 python tools/stage_times.py c2 5 >> gpurun_out/pyr_${TAG}.txt 2>&1
done
timeout 120 python tools/stage_times.py c4 10 >> gpurun_out/pyr_${TAG}.txt 2>&1
cat gpurun_out/pyr_${TAG}.txt

# selective_tc timing experiments (C5): kernel time of variants that skip parts of the work
for spec in "noprep:SELTC_SKIP_PREP" "nopipe:SELTC_SKIP_PIPE" "nopipe_nohist:SELTC_SKIP_PIPE,SELTC_NO_HIST" "nopipe_noload:SELTC_SKIP_PIPE,SELTC_NO_LOAD" "nopipe_none:SELTC_SKIP_PIPE,SELTC_NO_LOAD,SELTC_NO_HIST"; do
  name=${spec%%:*}; defs=${spec#*:}
  python paper_1508_01292_b200/build.py $name $defs > /dev/null 2>&1
  CCNN_LIB_VARIANT=$name timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:selective_cnn2 -c 1 python tools/stage_times.py c5 1 2>&1 | grep -E "duration|pct" | sed "s/^/$name /"
done

# Environment-knob A/B runs on the GPU box (no rebuild): each argument is a
# space-separated list of VAR=value settings; prints tools/setup_sweep.py's
# median phases for each. gpurun -- 'bash tools/tune_env.sh "" "CUTBDDC_LEAF=64" ...'
out=gpurun_out/tune_env.txt
mkdir -p gpurun_out
: > $out
for v in "$@"; do
  echo "== ${v:-default}" >> $out
  env $v timeout 600 python tools/setup_sweep.py ${TUNE_WORKLOAD:-cfg4} ${TUNE_REPS:-8} >> $out 2>&1
done
cat $out

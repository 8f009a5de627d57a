# DAG-kernel tuning on the GPU box: rebuild dense_dag.cu with each variant's
# CUTBDDC_SWEEP_* macros, run a short cfg4 bench, print the phases and the
# apply's solve-sweep time. Restores the default build at the end.
#   gpurun -- 'bash tools/tune_sweep.sh "-DCUTBDDC_SWEEP_FWD_ROWS=64" ...'
out=gpurun_out/tune.txt
mkdir -p gpurun_out
: > $out
run() {
  touch paper_1703_06323_b200/csrc/dense_dag.cu
  CUTBDDC_NVCC_EXTRA="$1" python -m paper_1703_06323_b200.build > /dev/null || { echo "$1 BUILD FAILED" >> $out; return; }
  timeout 300 python bench.py --no-cpu-baseline --no-cfg5 --workload ${TUNE_WORKLOAD:-cfg4} --steps ${TUNE_STEPS:-10} --warmup 3 2> /dev/null | python -c "
import json, sys
l = [x for x in sys.stdin if x.startswith('{')]
if not l: print('$1', 'NO OUTPUT'); sys.exit()
j = json.loads(l[-1]); ph = j['phases_ms']
print('%-70s it=%d asm=%.3f setup=%.3f pcg=%.3f sweeps=%.4f value=%.0f e2e=%.0f' % ('$1' or 'default', j['iterations'], ph['assembly'], ph['setup'], ph['pcg'], j['roofline']['launch_ms'], j['value'], j['e2e']['value']))
" >> $out
}
run ""
for v in "$@"; do run "$v"; done
run ""
cat $out

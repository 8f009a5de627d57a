# Multi-RHS width of the coarse-basis forward sweeps (H = L^{-1} C^T): rebuild
# with each -DCUTBDDC_MULTI_RHS=n and print the setup time and the H passes.
out=gpurun_out/tune_multi.txt
: > $out
run() {
  touch paper_1703_06323_b200/csrc/factor.cuh
  CUTBDDC_NVCC_EXTRA="$1" python -m paper_1703_06323_b200.build > /dev/null || { echo "$1 BUILD FAILED" >> $out; return; }
  CUTBDDC_PROFILE=1 timeout 300 python bench.py --no-cpu-baseline --no-cfg5 --no-batch --steps 10 --warmup 3 2> gpurun_out/tm.err | python -c "
import json, sys
l = [x for x in sys.stdin if x.startswith('{')]
j = json.loads(l[-1]); ph = j['phases_ms']
print('%-40s it=%d asm=%.3f setup=%.3f pcg=%.3f value=%.0f' % ('$1' or 'default', j['iterations'], ph['assembly'], ph['setup'], ph['pcg'], j['value']))
" >> $out
  grep -E "coarse basis H passes" gpurun_out/tm.err | tail -1 >> $out
}
run ""
for v in "$@"; do run "$v"; done
touch paper_1703_06323_b200/csrc/factor.cuh
python -m paper_1703_06323_b200.build > /dev/null
cat $out

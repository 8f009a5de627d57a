# Sweep-kernel variants at a large workload (default cfg5): rebuild sweep.cu
# with each variant's CUTBDDC_SWEEP_* macros and time one apply's solve
# sweeps (roofline hook). Restores the default build at the end.
#   gpurun -- 'bash tools/tune_sweep_cfg5.sh cfg5 "-DCUTBDDC_SWEEP_SLOTS=3" ...'
w=$1; shift
out=gpurun_out/tune_$w.txt
: > $out
run() {
  touch paper_1703_06323_b200/csrc/sweep.cu
  CUTBDDC_NVCC_EXTRA="$1" python -m paper_1703_06323_b200.build > /dev/null || { echo "$1 BUILD FAILED" >> $out; return; }
  timeout 600 python -c "
import sys; sys.path.insert(0, '.')
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get('$w'); s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
x, rep = s.pcg(rtol=cfg.rtol)
rf = s.roofline(reps=3)
print('%-50s sweeps %.3f ms  %.0f GB/s  pcg %.1f ms' % ('$1' or 'default', 1e3 * rf['seconds'], rf['bytes'] / rf['seconds'] / 1e9, 1e3 * rep['t_pcg']))
" >> $out 2>&1
}
run ""
for v in "$@"; do run "$v"; done
touch paper_1703_06323_b200/csrc/sweep.cu
python -m paper_1703_06323_b200.build > /dev/null
cat $out

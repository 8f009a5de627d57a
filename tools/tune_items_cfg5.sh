# Item-size variants (CUTBDDC_SWEEP_ITEMS=fwd_cols,bwd_cols,small_work) at one
# workload: one setup per variant, the apply's solve sweeps timed (roofline hook)
#   gpurun -- 'bash tools/tune_items_cfg5.sh cfg5 "256,32,32768" "128,32,32768" ...'
w=$1; shift
out=gpurun_out/tune_items_$w.txt
: > $out
for v in "$@"; do
  CUTBDDC_SWEEP_ITEMS="$v" timeout 600 python -c "
import sys; sys.path.insert(0, '.')
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get('$w'); s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
rf = s.roofline(reps=5)
print('%-20s sweeps %.3f ms  %.0f GB/s' % ('$v', 1e3 * rf['seconds'], rf['bytes'] / rf['seconds'] / 1e9))
" >> $out 2>&1
done
cat $out

# Sweep item-size A/B on the GPU box (no rebuild): for each CUTBDDC_SWEEP_ITEMS
# value "fwd_cols,bwd_cols", the apply's solve-sweep time (roofline hook).
#   gpurun -- 'bash tools/tune_items.sh cfg4 "" "128,16" "64,8"'
w=$1; shift
for v in "$@"; do
  CUTBDDC_SWEEP_ITEMS=$v timeout 300 python -c "
import sys; sys.path.insert(0, '.')
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get('$w'); s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
s.pcg(rtol=cfg.rtol)
rf = s.roofline(reps=5)
print('%-10s %-8s sweeps %.4f ms  %.0f GB/s' % ('$w', '${v:-auto}', 1e3 * rf['seconds'], rf['bytes'] / rf['seconds'] / 1e9))
"
done

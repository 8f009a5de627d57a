# Sweep ring A/B (no rebuild): CUTBDDC_SWEEP_RING=slot_doubles,bwd_rows values.
#   gpurun -- 'bash tools/tune_ring.sh cfg4 "3584,110" "5120,158"'
w=$1; shift
for v in "$@"; do
  CUTBDDC_SWEEP_RING=$v timeout 300 python -c "
import sys; sys.path.insert(0, '.')
from paper_1703_06323_b200 import configs, cutbddc as cb
cfg = configs.get('$w'); s = cb.GpuSolver(0); pb = cb.prepare(s, cfg); s.setup_bddc(pb.objects, cfg.weighting)
x, rep = s.pcg(rtol=cfg.rtol)
x, rep = s.pcg(rtol=cfg.rtol)
rf = s.roofline(reps=5)
print('%-10s %-10s sweeps %.4f ms  %.0f GB/s  pcg %.3f ms it %d' % ('$w', '$v', 1e3 * rf['seconds'], rf['bytes'] / rf['seconds'] / 1e9, 1e3 * rep['t_pcg'], rep['iterations']))
"
done

# A/B of k_coarse_out on one box: plain (one zc row per warp at a time, no H
# prefetch) against the default (four rows in flight + L2 prefetch of the
# block's H columns); per-iteration and per-apply times from tools/time_parts.py.
for round in 1 2; do
  for v in "-DCUTBDDC_COARSE_OUT_PLAIN" ""; do
    touch paper_1703_06323_b200/csrc/bddc.cu
    CUTBDDC_NVCC_EXTRA="$v" python -c "from paper_1703_06323_b200 import build; build.build()" || exit 1
    echo "== round $round flags '$v'"
    timeout 300 python tools/time_parts.py cfg4 2>&1 | tail -2
  done
done

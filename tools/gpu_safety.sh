# compute-sanitizer memcheck / racecheck / synccheck over small solves (the
# persistent dataflow kernels spin on completion counters: a missing fence or
# an out-of-bounds descriptor shows up here), then the BASELINE cfg5 runs that
# the bench does not cover. Logs go to gpurun_out/.
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in "cfg1" "cfg2 weighting=stiffness objects=cef"; do
    tag=$(echo "$tool $case" | tr ' =' '__')
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_case.py $case \
      > gpurun_out/san_$tag.log 2>&1; echo "$tool $case rc=$?" | tee -a gpurun_out/san_summary.txt
    tail -3 gpurun_out/san_$tag.log
  done
done
timeout 900 python tools/run_config.py cfg5 weighting=topological objects=ce > gpurun_out/cfg5_topo_ce.log 2>&1; echo "cfg5 topo ce rc=$?"
timeout 900 python tools/run_config.py cfg5 variant=v2 > gpurun_out/cfg5_v2.log 2>&1; echo "cfg5 v2 rc=$?"
cat gpurun_out/san_summary.txt gpurun_out/cfg5_*.log

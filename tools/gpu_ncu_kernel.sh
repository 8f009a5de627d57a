# ncu --set full of one kernel (regex $1) launched by `python $2 ...`; skip $3 launches
export PATH=/usr/local/cuda/bin:$PATH
k=$1; shift; script=$1; shift; skip=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
  -o gpurun_out/ncu_$k -f python $script "$@" > gpurun_out/ncu_$k.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu_$k.ncu-rep --page details --csv > gpurun_out/ncu_${k}_details.csv 2>/dev/null
grep -E "Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Registers Per|Theoretical Occ|Warp Cycles Per Issued|Eligible Warps|L1/TEX Hit|L2 Hit|Compute \(SM\) Throughput|Issue Slots Busy" gpurun_out/ncu_${k}_details.csv | cut -c1-200 | head -30

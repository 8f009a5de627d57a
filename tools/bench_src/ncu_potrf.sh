export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --import-source on --warp-sampling-interval 0 --kernel-name-base function -k regex:k_bench -c 1 -o gpurun_out/potrf_bench -f ./tools/bench_src/potrf_bench > gpurun_out/ncu_pb.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_pb.log

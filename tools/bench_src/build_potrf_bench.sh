# builds gpurun_out/potrf_bench (links the rest of the library from libcutbddc.so)
NCCLI=$(python -c "from paper_1703_06323_b200 import build; print(build.NCCL)")/include
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Ipaper_1703_06323_b200/csrc -Iinclude -I$NCCLI \
  tools/bench_src/potrf_bench.cu -o tools/bench_src/potrf_bench -Lpaper_1703_06323_b200 -lcutbddc \
  -Xlinker -rpath=\$ORIGIN/../../paper_1703_06323_b200

# Build the microbenchmarks from source (binaries are not committed):
#   tools/bin/mixbench    -- issue rate of the shipped fill instruction mix (DESIGN 5.2)
#   tools/bin/pipebench   -- which pipe each max/add form issues to (DESIGN 5.2)
#   tools/bin/hostpack_bench -- host 2-bit packing throughput (DESIGN 5.5)
set -e
cd "$(dirname "$0")"
mkdir -p bin
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3"
$NV -o bin/mixbench mixbench.cu
$NV -o bin/pipebench pipebench.cu
g++ -O3 -march=native -pthread -o bin/hostpack_bench hostpack_bench.cpp
$NV -o bin/dpx_latency dpx_latency.cu

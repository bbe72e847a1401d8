#!/bin/bash
# Build the instruction-throughput probe from source (the binary is not tracked) and run it on the
# GPU box: tools/microbench/run.sh > profiles/<round>_opbench.txt
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o "$HERE/opbench" "$HERE/opbench.cu"
"$HERE/opbench"

#!/bin/bash
# Build the issue-rate microbenchmark (tools/micro/pipes.cu) for sm_100a.
set -e
cd "$(dirname "$0")"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo pipes.cu -o pipes

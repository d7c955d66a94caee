#!/bin/bash
# phase traces of the three tick kernels (K1, append core, rank-1 core): trace build on the box
mkdir -p gpurun_out
export ISVD_NVCC_FLAGS=-DISVD_R1_TRACE
timeout 600 python -m paper_2605_24514_b200.build --force > gpurun_out/trace_build.log 2>&1 || exit 1
for B in 4096 512; do
  for G in 4 1; do
    timeout 300 python tools/k1_trace.py $B $G > gpurun_out/k1_trace_${B}_g$G.log 2>&1
  done
  timeout 300 python tools/r1_trace.py $B > gpurun_out/r1_trace_$B.log 2>&1
  timeout 300 python tools/r1_trace.py $B --arrow > gpurun_out/arrow_trace_$B.log 2>&1
done
tail -n 14 gpurun_out/k1_trace_*.log gpurun_out/r1_trace_*.log gpurun_out/arrow_trace_*.log

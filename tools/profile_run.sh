#!/bin/bash
# GPU profiling run for round artefacts (run under gpurun, one GPU).  Each ncu
# command runs only after the same command exited 0 without ncu.
#   gpurun_out/bench_full.json   default bench line (plain run, no profiler)
#   gpurun_out/launches.csv      ncu launch list (gpu__time_duration) of a short bench
#   gpurun_out/<k>.ncu-rep       ncu --set full of the dominant kernels
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
SHORT="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
$SHORT > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1
FULL="ncu --set full --clock-control none --import-source on"
$FULL -k regex:rotate_reg_kernel -s 40 -c 1 -o gpurun_out/rot5a $SHORT > gpurun_out/ncu_rot.log 2>&1
$FULL -k regex:jacobi32 -s 4 -c 1 -o gpurun_out/jacobi32 $SHORT > gpurun_out/ncu_j32.log 2>&1
$FULL -k regex:"arrow_svd" -s 4 -c 1 -o gpurun_out/arrow40 $SHORT > gpurun_out/ncu_arrow.log 2>&1
$FULL -k regex:project_append -s 4 -c 1 -o gpurun_out/proj5a $SHORT > gpurun_out/ncu_proj.log 2>&1
# config 5b (k = 128): the deferred-U flush rotation (DMMA) and the cluster arrow core
python tools/time_5b.py > gpurun_out/time5b.log 2>&1 && \
$FULL -k regex:"rotate_kernel" -c 1 -s 5 -o gpurun_out/rot5b_flush python tools/time_5b.py > gpurun_out/ncu_rot5b.log 2>&1
$FULL -k regex:"arrow_svd" -c 1 -s 4 -o gpurun_out/arrow129 python tools/time_5b.py 262144 > gpurun_out/ncu_arrow129.log 2>&1
ls -la gpurun_out

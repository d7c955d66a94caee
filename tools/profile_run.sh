#!/bin/bash
# GPU profiling run for round artefacts (run under gpurun).  Produces:
#   gpurun_out/bench_full.json      default bench line (plain run, no profiler)
#   gpurun_out/launches.csv         ncu launch list (gpu__time_duration) of a short bench
#   gpurun_out/rot.ncu-rep          ncu --set full of the rotation kernel
#   gpurun_out/core.ncu-rep         ncu --set full of the two core-SVD kernels
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
SHORT="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4"
$SHORT > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1
$SHORT > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rotate_kernel -s 6 -c 1 -o gpurun_out/rot $SHORT > gpurun_out/ncu_rot.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi32|arrow_svd" -s 4 -c 2 -o gpurun_out/core $SHORT > gpurun_out/ncu_core.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:project_append -s 2 -c 1 -o gpurun_out/proj $SHORT > gpurun_out/ncu_proj.log 2>&1
ls -la gpurun_out

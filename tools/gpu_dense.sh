#!/bin/bash
# Dense contractions of the refresh / oracle / metrics path at config 4's
# final size: timing, ncu --set full of one launch per kernel, launch list.
# (compute-sanitizer is closed on this GPU pool.)
mkdir -p gpurun_out
timeout 900 python tools/dense_kernels.py > gpurun_out/dense_kernels.json 2> gpurun_out/dense_kernels.err || exit 1
FULL="timeout 900 ncu --set full --clock-control none --import-source on"
$FULL -k regex:frob_tile -c 1 -o gpurun_out/frob_tile python tools/dense_kernels.py --once > gpurun_out/ncu_frob.log 2>&1
$FULL -k regex:dsvd_round -s 40 -c 1 -o gpurun_out/dsvd_round python tools/dense_kernels.py --once > gpurun_out/ncu_dsvd.log 2>&1
$FULL -k regex:gram_tile -c 1 -o gpurun_out/gram_tile python tools/dense_kernels.py --once > gpurun_out/ncu_gram.log 2>&1
$FULL -k regex:gemm_tile -c 1 -o gpurun_out/gemm_tile python tools/dense_kernels.py --once > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_launches.csv python tools/dense_kernels.py --once > gpurun_out/ncu_dense_launch.log 2>&1
ls -la gpurun_out

#!/bin/bash
# Round artefacts on one GPU: GPU tests, smoke, default bench line, reference
# arm, ncu launch list of the timed 5a ticks, ncu --set full of the tick
# kernels (each ncu run only after the same command exited 0 without ncu),
# per-GPU shares of 5a (512 / 1024 / 2048 streams) and single-stream latencies.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
SHORT="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1
FULL="timeout 600 ncu --set full --clock-control none --kernel-name-base demangled"
for spec in "project_append32:proj5a:8" "rank1_fast:r1fast:8" "arrow_cta:arrowcta:8" "rotate_reg_kernel<.int.40:vflush5a:0" "rotate_reg_kernel<.int.32, .bool.0>:flush5a:0"; do
  IFS=: read k name sk <<< "$spec"
  $FULL -k "regex:$k" -s $sk -c 1 -o gpurun_out/$name $SHORT > gpurun_out/ncu_$name.log 2>&1
done
# config 5b kernels: the final deferred-U flush (rotate_kernel<128>) and the three tick kernels
T5="python tools/time_5b.py"
timeout 300 $T5 > gpurun_out/time_5b.log 2>&1
for spec in "rotate_kernel<.int.128:rot5b_flush:0" "proj_cluster_reg:proj5b:20" "arrow_svd_kernel<.int.136:arrow5b:20" "rotate_nsplit:rot5b_tick:20"; do
  IFS=: read k name sk <<< "$spec"
  $FULL -k "regex:$k" -s $sk -c 1 -o gpurun_out/$name $T5 > gpurun_out/ncu_$name.log 2>&1
done
for B in 512 1024 2048; do
  timeout 300 python tools/exp5a.py --streams $B --groups 1,2,4 > gpurun_out/exp5a_$B.log 2>&1
done
timeout 600 python tools/b1_breakdown.py > gpurun_out/b1_breakdown.log 2>&1
# summaries written on the box (the reports with source exceed the 64 MiB merge limit)
ISVD_SUMMARY_OUT=gpurun_out python tools/ncu_summary.py round > gpurun_out/ncu_summary.log 2>&1
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
cp /tmp/ncu_reps/proj5a.ncu-rep /tmp/ncu_reps/r1fast.ncu-rep /tmp/ncu_reps/arrowcta.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
ls -la gpurun_out

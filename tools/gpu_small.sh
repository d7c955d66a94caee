#!/bin/bash
# small-batch tick rates (per-GPU shares of 5a at 2/4/8 GPUs) and single-stream latency
mkdir -p gpurun_out
for sN in 2048 1024 512; do
  timeout 600 python tools/exp5a.py --streams $sN --ticks 256 --groups 1,2,4 > gpurun_out/exp5a_$sN.log 2>&1
  tail -4 gpurun_out/exp5a_$sN.log
done
timeout 600 python tools/b1_breakdown.py > gpurun_out/b1_breakdown.json 2> gpurun_out/b1_breakdown.err; cat gpurun_out/b1_breakdown.json
timeout 900 python tools/latency_cfgs.py 300 > gpurun_out/latency_cfgs.json 2> gpurun_out/latency_cfgs.err; cat gpurun_out/latency_cfgs.json

#!/bin/bash
# core-kernel check: [parity / engine tests,] short bench, then phase traces (trace build)
# QUICK=1 skips the tests
mkdir -p gpurun_out
if [ "${QUICK:-0}" != "1" ]; then
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_vdefer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_core.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_core.log
tail -n 5 gpurun_out/pytest_core.log
fi
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 64 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err
python tools/summarize_bench.py gpurun_out/short.json 2>/dev/null | head -8
export ISVD_NVCC_FLAGS="-DISVD_R1_TRACE -DISVD_ARROW_STATS"
timeout 600 python -m paper_2605_24514_b200.build --force > gpurun_out/trace_build.log 2>&1 || exit 1
for B in 4096 512; do
  timeout 300 python tools/r1_trace.py $B > gpurun_out/r1_trace_$B.log 2>&1
  timeout 300 python tools/r1_trace.py $B --arrow > gpurun_out/arrow_trace_$B.log 2>&1
done
tail -n 14 gpurun_out/arrow_trace_*.log gpurun_out/r1_trace_*.log

#!/bin/bash
# projection-kernel check: parity / engine tests, short bench, then K1 phase trace (trace build)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_vdefer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_k1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k1.log
tail -n 5 gpurun_out/pytest_k1.log
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 64 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err
python tools/summarize_bench.py gpurun_out/short.json 2>/dev/null | head -30
export ISVD_NVCC_FLAGS=-DISVD_R1_TRACE
timeout 600 python -m paper_2605_24514_b200.build --force > gpurun_out/trace_build.log 2>&1 || exit 1
for B in 4096 512; do
  timeout 300 python tools/k1_trace.py $B 4 > gpurun_out/k1_trace_${B}_g4.log 2>&1
done
tail -n 12 gpurun_out/k1_trace_*_g4.log

#!/bin/bash
# projection-kernel check: [parity / engine tests,] short bench, ncu of K1, then K1 phase trace (trace build)
# QUICK=1 skips the tests, NCU=0 the ncu capture
mkdir -p gpurun_out
if [ "${QUICK:-0}" != "1" ]; then
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_vdefer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_k1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k1.log
tail -n 5 gpurun_out/pytest_k1.log
fi
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 64 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err
python tools/summarize_bench.py gpurun_out/short.json 2>/dev/null | head -8
if [ "${NCU:-1}" = "1" ]; then
NS="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_append32 -s 6 -c 1 -o gpurun_out/k1p32 $NS > gpurun_out/ncu_k1p32.log 2>&1
tail -n 2 gpurun_out/ncu_k1p32.log
fi
export ISVD_NVCC_FLAGS=-DISVD_R1_TRACE
timeout 600 python -m paper_2605_24514_b200.build --force > gpurun_out/trace_build.log 2>&1 || exit 1
for B in 4096 512; do
  for G in 4 1; do
  timeout 300 python tools/k1_trace.py $B $G > gpurun_out/k1_trace_${B}_g$G.log 2>&1
  done
done
tail -n 12 gpurun_out/k1_trace_*.log

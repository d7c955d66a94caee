timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vdefer.py -m gpu -q -p no:cacheprovider -k "append or row or cfg5a or golden or mixed or lazy or vdefer or trajectory" > gpurun_out/pytest_arrow.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_arrow.log; tail -3 gpurun_out/pytest_arrow.log
bash tools/gpu_quick.sh 2>&1 | grep -v "Broken\|Traceback\|File\|print"
ISVD_NVCC_FLAGS=-DISVD_R1_TRACE python -m paper_2605_24514_b200.build --force > /dev/null && python tools/r1_trace.py 4096 --arrow

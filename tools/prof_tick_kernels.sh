mkdir -p gpurun_out
SHORT="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1 || exit 1
FULL="timeout 600 ncu --set full --clock-control none --import-source on"
for spec in "jacobi32c:jacobi32:8" "arrow_svd:arrow40:8" "project_append:proj5a:8"; do
  IFS=: read k name sk <<< "$spec"
  $FULL -k regex:$k -s $sk -c 1 -o gpurun_out/$name $SHORT > gpurun_out/ncu_$name.log 2>&1
done
ls -la gpurun_out

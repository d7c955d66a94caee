#!/bin/bash
# quick A/B: short 5a bench (device ticks), launch list of 16 timed ticks
mkdir -p gpurun_out
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 32 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err || { tail -20 gpurun_out/short.err; exit 1; }
NS="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $NS > gpurun_out/ncu_launch.log 2>&1
python tools/launch_stats.py gpurun_out/launches.csv | head -8
python -c "
import json
d=json.loads(open('gpurun_out/short.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'])
for k,v in d['kernels'].items(): print('  ',k, round(v['ms_per_step']*1000,1),'us')
"

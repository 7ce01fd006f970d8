#!/bin/bash
# K2 on 36 SMs (the two-stream share in config 3): per-SM rate + one ncu --set full capture with
# source counters (stall reasons per SASS line) for the decode kernel.
mkdir -p gpurun_out
for n in 36 148; do
PATTN_DECODE_SMS=$n timeout 200 python bench.py --workload c3d_decode_part --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['kernel_ms']['decode']; print('decode on $n SMs', round(t*1e3,1), 'us', round(0.9407/t,1), 'GB/s total', round(0.9407/t/$n*1e3,1), 'GB/s/SM')"
done
PATTN_DECODE_SMS=36 timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k2_decode" -s 3 -c 1 -o gpurun_out/k2_sm36 -f python bench.py --workload c3d_decode_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
ls -la gpurun_out/k2_sm36.ncu-rep

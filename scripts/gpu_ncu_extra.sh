#!/bin/bash
# Extra ncu --set full captures: K2 and K3 on config 4 (long-context decode).
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k2_decode" -s 3 -c 1 -o gpurun_out/k2_c4_full -f \
    python bench.py --workload c4_decode128k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k3_reduce" -s 3 -c 1 -o gpurun_out/k3_c4_full -f \
    python bench.py --workload c4_decode128k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/*_c4_full.ncu-rep

#!/bin/bash
# Quick GPU pass: smoke, bench lines for configs 2-4, ncu launch lists of our kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
python bench.py --workload c2_decode8b --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
python bench.py --workload c4_decode128k --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err
for c in c2_decode8b c4_decode128k c3_mixed8b; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k[1-5]_" -c 20 --csv --log-file gpurun_out/ncu_$c.csv \
      python bench.py --workload $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cat gpurun_out/bench_c*.json

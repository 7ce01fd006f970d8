#!/bin/bash
# Quick GPU pass: smoke, bench lines for configs 2-4, ncu launch lists of our kernels,
# one ncu --set full capture of the prefill kernel.  Every step is time-bounded.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -2 gpurun_out/bench_c3.err
timeout 200 python bench.py --workload c2_decode8b --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err
timeout 200 python bench.py --workload c4_decode128k --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
for c in c2_decode8b c4_decode128k c3_mixed8b; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k[1-5]_" -c 20 --csv --log-file gpurun_out/ncu_$c.csv \
      python bench.py --workload $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k1_prefill" -s 2 -c 1 -o gpurun_out/k1_c3_full -f \
    python bench.py --workload c3_mixed8b --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1_full.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k2_decode" -s 3 -c 1 -o gpurun_out/k2_c2_full -f \
    python bench.py --workload c2_decode8b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_c*.csv
for f in gpurun_out/bench_c*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['config']['workload'], 'value %.0f tok/s' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})
for k,v in d['roofline_kernels'].items(): print('   ', k, round(v['achieved'],1), v['unit'], 'frac', round(v['frac'],3))
print('   e2e', d['e2e'] and round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],1), 'clocks', d['clocks'])
"; done

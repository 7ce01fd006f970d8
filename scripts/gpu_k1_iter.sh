#!/bin/bash
# K1 iteration loop: prefill parity tests + c3 bench line + launch list.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or random_mixed or chunked or needle" 2>&1 | tail -3
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -2 gpurun_out/bench_c3.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1])
print(d['config']['workload'], 'value %.0f tok/s' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})
for k,v in d['roofline_kernels'].items(): print('   ', k, round(v['achieved'],1), v['unit'], 'frac', round(v['frac'],3))
"
if [ "$1" == "full" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k1_prefill" -s 2 -c 1 -o gpurun_out/k1_c3_full -f \
    python bench.py --workload c3_mixed8b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k1_full.log 2>&1
fi

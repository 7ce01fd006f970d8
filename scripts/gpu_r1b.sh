#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_write_kv.py -x -q 2>&1 | tail -5
summ() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['config']['workload'], d['config']['parallelism'], 'value %.0f tok/s' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})
for k,v in d['roofline_kernels'].items(): print('   ', k, round(v['achieved'],1), v['unit'], 'frac', round(v['frac'],3))
print('   graph', d['cuda_graph'], 'e2e', d['e2e'] and round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'])
"; }
timeout 200 python bench.py --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_c3_s1.json 2>gpurun_out/b_c3_s1.err; summ gpurun_out/b_c3_s1.json
timeout 300 python bench.py --workload c5_mixed70b --steps 20 --warmup 5 > gpurun_out/b_c5.json 2>gpurun_out/b_c5.err; summ gpurun_out/b_c5.json; tail -3 gpurun_out/b_c5.err
for m in seq kvhead; do
timeout 200 python bench.py --workload c5_mixed70b --shard $m --sim-world 8 --sim-rank 0 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_c5_$m.json 2>gpurun_out/b_c5_$m.err; summ gpurun_out/b_c5_$m.json; tail -3 gpurun_out/b_c5_$m.err
done

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
bash scripts/gpu_bench_quick.sh
timeout 300 python bench.py --workload c5_mixed70b --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err
for m in seq kvhead; do
timeout 200 python bench.py --workload c5_mixed70b --shard $m --sim-world 8 --sim-rank 0 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5_${m}8_rank0.json 2>/dev/null
done
for f in gpurun_out/bench_c5*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'value %.0f tok/s' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, d['config']['parallelism'])
"; done

#!/bin/bash
# Exercise bench.py's multi-rank path (torchrun, 2 ranks) on a 1-GPU box: gloo, both ranks on GPU 0.
export PATTN_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 300 $R bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err; echo "weak rc=$?"; tail -c 400 gpurun_out/mr_weak.json
timeout 300 $R bench.py --gpus 2 --workload c5_mixed70b --shard seq --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_seq.json 2> gpurun_out/mr_seq.err; echo "seq rc=$?"; tail -c 300 gpurun_out/mr_seq.json
timeout 300 $R bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"; tail -c 200 gpurun_out/mr_ref.json
grep -i -E "error|Traceback" gpurun_out/mr_*.err | head -10

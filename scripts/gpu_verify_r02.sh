#!/bin/bash
# Round-2 verification pass on the final tree: GPU tests, smoke, every bench line, the launch
# list of the default bench command.
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; tail -3 gpurun_out/final/smoke.txt
timeout 600 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; tail -1 gpurun_out/final/bench_default.err
for W in c2_decode8b c4_decode128k c5_mixed70b c3p_prefill_part x_g7_mixed x_d64_mixed x_bs7_decode32k; do
  ST=2; [ $W == c3p_prefill_part ] && ST=1
  timeout 300 python bench.py --workload $W --streams $ST --steps 50 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/final/bench_$W.json 2> gpurun_out/final/bench_$W.err
done
timeout 300 python bench.py --workload c1_tiny --steps 100 --warmup 10 --no-sub > gpurun_out/final/bench_c1_tiny.json 2> gpurun_out/final/bench_c1_tiny.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k[1-7]_" -c 120 --csv --log-file gpurun_out/final/ncu_default_command.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out/final

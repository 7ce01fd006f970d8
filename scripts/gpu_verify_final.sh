#!/bin/bash
# Final pass: GPU tests, smoke, default bench line + the widened-envelope lines, default-command launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for W in ${WS:-x_bs7_mixed x_bs7_decode32k}; do
  timeout 300 python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k[1-7]w?_" -c 120 --csv --log-file gpurun_out/ncu_default_command.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_default_command.csv

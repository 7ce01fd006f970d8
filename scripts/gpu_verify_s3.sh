#!/bin/bash
# Final verification pass of the tree (round 2, session 3): GPU tests, smoke, every bench line,
# ncu launch lists (default command + per config), ncu --set full of K1 (config 3's prefill part)
# and K2W (configs 2 and 4, and on 36 SMs), the K1 tensor-pipe counters, the 2-rank functional run.
# Outputs in gpurun_out/ (flat: scripts/profile_summary.py r02 copies them into profiles/r02).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.err
for W in c2_decode8b c4_decode128k c5_mixed70b c3p_prefill_part x_g7_mixed x_d64_mixed x_bs7_decode32k; do
  ST=2; [ $W == c3p_prefill_part ] && ST=1
  timeout 300 python bench.py --workload $W --streams $ST --steps 50 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 300 python bench.py --workload c1_tiny --steps 100 --warmup 10 --no-sub > gpurun_out/bench_c1_tiny.json 2> gpurun_out/bench_c1_tiny.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k[1-7]w?_" -c 120 --csv --log-file gpurun_out/ncu_default_command.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
for c in c2_decode8b c4_decode128k c3_mixed8b c3p_prefill_part; do
  ST=2; [ $c == c3p_prefill_part ] && ST=1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k[1-5]w?_" -c 20 --csv --log-file gpurun_out/ncu_$c.csv \
      python bench.py --workload $c --streams $ST --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"k1_prefill" -s 2 -c 1 --csv --log-file gpurun_out/ncu_k1_tensor.csv \
    python bench.py --workload c3p_prefill_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k1_prefill" -s 2 -c 1 -o gpurun_out/k1_c3p_full -f \
    python bench.py --workload c3p_prefill_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
for c in c2_decode8b c4_decode128k; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k2w_decode" -s 3 -c 1 -o gpurun_out/k2w_${c:0:2}_full -f \
      python bench.py --workload $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
done
PATTN_DECODE_SMS=36 timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k2w_decode" -s 3 -c 1 -o gpurun_out/k2w_sm36_main -f \
    python bench.py --workload c3d_decode_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
export PATTN_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 $R bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err; echo "multirank rc=$?"
ls gpurun_out/*.ncu-rep

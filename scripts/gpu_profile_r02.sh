#!/bin/bash
# Round-2 GPU pass: smoke, bench lines (default + per workload), ncu launch lists, the K1
# tensor-pipe metrics, ncu --set full captures of K1 and K2, the multi-rank functional check.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -2 gpurun_out/bench_default.err
for W in c2_decode8b c4_decode128k c5_mixed70b c3p_prefill_part x_g7_mixed x_d64_mixed x_bs7_decode32k; do
  ST=2; [ $W == c3p_prefill_part ] && ST=1
  timeout 300 python bench.py --workload $W --streams $ST --steps 50 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; tail -1 gpurun_out/bench_$W.err
done
timeout 300 python bench.py --workload c1_tiny --steps 100 --warmup 10 --no-sub > gpurun_out/bench_c1_tiny.json 2> gpurun_out/bench_c1_tiny.err
# launch lists (cold-cache, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k[1-7]_" -c 120 --csv --log-file gpurun_out/ncu_default_command.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
for c in c2_decode8b c4_decode128k c3_mixed8b c3p_prefill_part; do
  ST=2; [ $c == c3p_prefill_part ] && ST=1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k[1-5]_" -c 20 --csv --log-file gpurun_out/ncu_$c.csv \
      python bench.py --workload $c --streams $ST --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
done
# K1 tensor-pipe counters (reconciled against the flop-derived fraction in profiles/r02/summary.txt)
timeout 300 ncu --metrics gpu__time_duration.sum,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg \
    --clock-control none -k regex:"k1_prefill" -s 2 -c 1 --csv --log-file gpurun_out/ncu_k1_tensor.csv \
    python bench.py --workload c3p_prefill_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k1_prefill" -s 2 -c 1 -o gpurun_out/k1_c3p_full -f \
    python bench.py --workload c3p_prefill_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k2_decode" -s 3 -c 1 -o gpurun_out/k2_c4_full -f \
    python bench.py --workload c4_decode128k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k2_decode" -s 3 -c 1 -o gpurun_out/k2_c2_full -f \
    python bench.py --workload c2_decode8b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
# multi-rank path (torchrun, 2 ranks, gloo, both on GPU 0): functional only, never a number
export PATTN_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 $R bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err; echo "multirank rc=$?"
timeout 300 $R bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "ref rc=$?"
ls gpurun_out/*.ncu-rep

#!/bin/sh
# Round-2 evidence refresh on one B200 (run under gpurun from the repo root):
# per config an ncu FP64-flop count and an ncu --set full capture of its kernel,
# the bench's launch list (gpu__time_duration, B200_PROFILING.md), then the bench.
set -u
mkdir -p gpurun_out
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__ops_path_tensor_src_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
for c in c1 c2 c3 c4 c5; do
  timeout 300 ncu --metrics $M --clock-control none --csv -c 1 python tools/prof_one.py $c 1 > gpurun_out/flops_$c.csv 2>/dev/null
  timeout 400 ncu --set full --import-source on --clock-control none -c 1 -f -o gpurun_out/full_$c python tools/prof_one.py $c 1 > gpurun_out/full_$c.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-parity --e2e-steps 0 > gpurun_out/ncu_bench.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
echo "bench rc=$?"

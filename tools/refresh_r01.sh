set -u
mkdir -p gpurun_out
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__ops_path_tensor_src_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
for c in c3 c5; do
  timeout 300 ncu --metrics $M --clock-control none --csv -c 1 python tools/prof_one.py $c 1 > gpurun_out/flops_$c.csv 2>/dev/null
  timeout 300 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/full_$c python tools/prof_one.py $c 1 > gpurun_out/full_$c.log 2>&1
done
bash tools/bench_all.sh

#!/bin/bash
# Runs bench.py for every config (ours + reference arm) and the ncu launch list
# of the default bench command; outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
  python bench.py --config $c --impl reference --steps 3 --warmup 1 >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
done
# launch list of the default bench command (cold, serialised; compare shares)
python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
echo done

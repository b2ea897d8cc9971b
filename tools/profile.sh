#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU):
#   bash tools/profile.sh <tag> [bench args...]
# 1. the bench line itself (no profiler attached);
# 2. the ncu launch list of the same bench command (gpu__time_duration per launch, cold/serialised);
# 3. one `ncu --set full` capture of the dominant SpMM launch (case 4 of the step: 768x3072 2:4).
# Outputs land in gpurun_out/<tag>_*; tools/ncu_summary.py turns them into profiles/.
tag=$1; shift
mkdir -p gpurun_out
timeout 600 python bench.py "$@" --out gpurun_out/${tag}_bench.jsonl > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 --no-graph --lanes 1 "$@" > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 12 -c 1 -o gpurun_out/${tag}_full \
   python bench.py --profile --steps 1 --warmup 1 --no-graph --lanes 1 "$@" > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full rc=$?"

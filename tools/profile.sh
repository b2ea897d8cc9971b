#!/bin/bash
# usage: bash scripts_profile.sh <tag> [bench args...]   (run under gpurun; writes gpurun_out/<tag>_*)
tag=$1; shift
mkdir -p gpurun_out
timeout 600 python bench.py "$@" --out gpurun_out/${tag}_bench.jsonl > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?"; tail -c 3000 gpurun_out/${tag}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 --no-graph "$@" > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 9 -c 3 -o gpurun_out/${tag}_full \
   python bench.py --profile --steps 1 --warmup 1 --no-graph "$@" > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -5 gpurun_out/${tag}_ncu_full.log

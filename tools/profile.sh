#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU):
#   bash tools/profile.sh <tag> [bench args...]
# 1. the bench line itself (no profiler attached), recording the per-case plans it used;
# 2. the ncu launch list of the same step with those plans (gpu__time_duration + DRAM bytes per
#    launch, cold/serialised: compare shares, not absolute times);
# 3. one `ncu --set full` capture of the dominant SpMM launch: case DOM (default 3, 768x3072 2:4
#    of C2), i.e. the (DOM+1)-th SpMM launch of the first warm-up step;
# 4. one `ncu --set full` capture of the tcgen05 kernel on C3 (1024x4096x16384 1:4, g = 64).
# Outputs land in gpurun_out/<tag>_*; tools/ncu_summary.py turns them into profiles/.
tag=$1; shift
DOM=${DOM:-3}
mkdir -p gpurun_out
timeout 900 python bench.py "$@" --plans-out gpurun_out/${tag}_plans.json --out gpurun_out/${tag}_bench.jsonl \
   > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/${tag}_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 --no-graph --lanes 1 --plans-in gpurun_out/${tag}_plans.json "$@" \
   > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s ${DOM} -c 1 -o gpurun_out/${tag}_full \
   python bench.py --profile --steps 1 --warmup 1 --no-graph --lanes 1 --plans-in gpurun_out/${tag}_plans.json "$@" \
   > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 0 -c 1 -o gpurun_out/${tag}_tc_full \
   python bench.py --config 2 --g 64 --profile --steps 1 --warmup 1 --no-graph --lanes 1 --no-tune \
   > gpurun_out/${tag}_ncu_tc_full.log 2>&1
echo "ncu tc full rc=$?"
# 5. one `ncu --set full` capture of the K1 sparsify launch of the dominant case
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparsify -s ${DOM} -c 1 -o gpurun_out/${tag}_sp_full \
   python bench.py --profile --steps 1 --warmup 1 --no-graph --lanes 1 --plans-in gpurun_out/${tag}_plans.json "$@" \
   > gpurun_out/${tag}_ncu_sp_full.log 2>&1
echo "ncu sparsify full rc=$?"
# export the full captures to CSV (raw metrics, details, per-instruction source) and drop the
# .ncu-rep files so gpurun_out/ stays under the 64 MiB copy-back limit
for r in full tc_full sp_full; do
  f=gpurun_out/${tag}_${r}.ncu-rep
  if [ -f $f ]; then
    ncu -i $f --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
    ncu -i $f --page details --csv > gpurun_out/${tag}_${r}_details.csv 2>/dev/null
    ncu -i $f --page source --csv --print-source sass > gpurun_out/${tag}_${r}_source.csv 2>/dev/null
    rm -f $f
  fi
done
ls -la gpurun_out/

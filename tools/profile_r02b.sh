#!/bin/bash
# Round-2 second profiling pass (one GPU, under gpurun), after the one-launch grouped sparsify:
# launch list of the bench step + full captures of the grouped SpMM and the grouped sparsify.
# Outputs gpurun_out/${TAG}_* (summarised by TAG=r02b tools/ncu_summary_r02.py).
TAG=${TAG:-r02b}
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 --no-graph > gpurun_out/${TAG}_launch_bench.log 2>&1
echo "launches rc=$?"
full() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
     -o gpurun_out/${TAG}_$name "$@" > gpurun_out/${TAG}_${name}.log 2>&1
  echo "$name rc=$?"
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page raw --csv > gpurun_out/${TAG}_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page details --csv > gpurun_out/${TAG}_${name}_details.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_$name.ncu-rep
}
full grouped spmm_simt_batched 1 python bench.py --profile --steps 1 --warmup 1 --no-graph
full gsparsify sparsify_grouped_nm_batched 1 python bench.py --profile --steps 1 --warmup 1 --no-graph

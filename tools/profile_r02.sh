#!/bin/bash
# Round-2 profiling (one GPU, under gpurun): launch list of the bench step + full captures of the
# dominant kernels.  Outputs: gpurun_out/r02_*.csv (summarised by tools/ncu_summary_r02.py).
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 --no-graph > gpurun_out/r02_launch_bench.log 2>&1
echo "launches rc=$?"
full() {  # name, kernel regex, skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
     -o gpurun_out/r02_$name "$@" > gpurun_out/r02_${name}.log 2>&1
  echo "$name rc=$?"
  ncu -i gpurun_out/r02_$name.ncu-rep --page raw --csv > gpurun_out/r02_${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_$name.ncu-rep --page details --csv > gpurun_out/r02_${name}_details.csv 2>/dev/null
  rm -f gpurun_out/r02_$name.ncu-rep
}
full grouped spmm_simt_batched 1 python bench.py --profile --steps 1 --warmup 1 --no-graph
full gsparsify sparsify_grouped_nm_batched 0 python bench.py --profile --steps 1 --warmup 1 --no-graph
full sp24 spmm_sp24 0 python tools/sp24_bench.py --config 2 --tiles 1 --reps 1
full sddmm sddmm 0 python -c "
import torch, sys; sys.path.insert(0, '.')
from paper_2304_07613_b200 import sten
W = torch.randn(3072, 768, device='cuda') * 0.02
v, i = sten.sparsify_grouped_nm(W, 2, 4, 4)
G = torch.randn(3072, 32768, device='cuda'); B = torch.randn(768, 32768, device='cuda')
sten.sddmm_grouped_nm(G, B, i, 2, 4, 4); torch.cuda.synchronize()"
full nmgx nmg_sparsify 0 python -c "
import torch, sys; sys.path.insert(0, '.')
from paper_2304_07613_b200 import sten
W = torch.randn(768, 3072, device='cuda') * 0.02
sten.nmg_sparsify(W, 2, 4, 4, method=2); torch.cuda.synchronize()"

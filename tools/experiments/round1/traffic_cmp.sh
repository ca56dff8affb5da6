#!/bin/bash
M="dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__cluster_dim_x,smsp__inst_executed.sum,l1tex__t_bytes.sum"
for s in k1 dx dw; do
  cat > /tmp/cb_$s.py <<PY
import torch
g=torch.Generator(device='cuda').manual_seed(0)
x=torch.randn(8192,4096,device='cuda',generator=g).to(torch.bfloat16)
w=(torch.randn(256000,4096,device='cuda',generator=g)*0.02).to(torch.bfloat16)
p=(torch.randn(8192,256000,device='cuda',generator=g)*4e-6).to(torch.bfloat16)
f={'k1':lambda: x@w.T, 'dx':lambda: p@w, 'dw':lambda: p.T@x}['$s']
for _ in range(3): f()
torch.cuda.synchronize()
PY
  timeout 300 ncu --metrics $M --clock-control none -k regex:"nvjet|gemm|cutlass|sm100" -s 2 -c 1 python /tmp/cb_$s.py 2>&1 | grep -E "^\s+(dram|lts|gpu__time|sm__cyc|launch|smsp|l1tex|  [a-z])|nvjet|Kernel" | sed "s/^/cublas $s /"
done
for k in "k1 0 1" "k1 0 2" "dx 16 1" "dx 16 2" "dw -16 1" "dw -4 2"; do
  set -- $k
  VP_NH=$3 timeout 120 ncu --metrics $M --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe $1 $2 0 0 1 2>&1 | grep -E "^\s+(dram|lts|gpu__time|sm__cyc|launch|smsp|l1tex)" | sed "s/^/ours $1 nh=$3 /"
done

#!/bin/bash
for k in "dw -4" "dx 16" "k1 0"; do set -- $k
  for b in gemm_probe_ls8 gemm_probe_ls32 gemm_probe; do
    echo "== $b $1"; VP_NH=2 timeout 60 ./tools/$b $1 $2 0 0 30 | grep -E "ideal|TFLOP" || continue
    VP_NH=2 timeout 60 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -s 1 -c 1 ./tools/$b $1 $2 0 0 1 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/   /"
  done
done

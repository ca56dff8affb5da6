#!/bin/bash
for k in "k1 0" "dx 16" "dw -4"; do
  set -- $k
  for nh in 1 2; do
    r=$2; if [ $1 = dw ] && [ $nh = 1 ]; then r=-16; fi
    VP_NH=$nh timeout 120 ./tools/gemm_probe $1 $r 0 0 60
  done
done
VP_NH=1 timeout 60 ./tools/gemm_probe sq8192 0 0 0 200

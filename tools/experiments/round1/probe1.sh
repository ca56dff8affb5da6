#!/bin/bash
# rasterisation / L2-policy sweep: sustained time (10 iters) + DRAM bytes (ncu, 1 launch)
P=./tools/gemm_probe
run() {
  timeout 60 $P "$@" 20
  timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 $P "$@" 1 2>/dev/null | grep -E "dram__bytes|hit_rate|duration" | awk '{print "   ", $1, $(NF-1), $NF}'
}
for r in 0 16 8 4; do run k1 $r -1 -1; done
run k1 8 0 0
run k1 0 0 0
for r in 8 4 16 32 -4; do run dx $r -1 -1; done
run dx 8 0 0
for r in -16 -8 16 0; do run dw $r -1 -1; done
run dw -16 0 0

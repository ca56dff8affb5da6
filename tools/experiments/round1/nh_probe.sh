#!/bin/bash
timeout 120 ./tools/gemm_selftest > gpurun_out/selftest_nh.log 2>&1; echo selftest_rc=$?; grep -E "FAIL|SELFTEST|nh=2" gpurun_out/selftest_nh.log | head -20
sample() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv & echo $!; }
summ() { python - "$1" <<'PY'
import sys, statistics
v=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
v=v[len(v)//4:]
print("   %s: clk median %.0f MHz  power median %.0f W (%d samples)" % (sys.argv[1], statistics.median(float(a) for a,b in v), statistics.median(float(b) for a,b in v), len(v)))
PY
}
for rep in 1 2; do
for k in "dx 16" "dx 8" "dw -16" "dw -8"; do
  set -- $k
  for nh in 1 2; do
    r=$2; if [ $nh = 2 ] && [ $1 = dw ]; then r=$(( $2 / 2 )); fi
    P=$(sample); VP_NH=$nh timeout 120 ./tools/gemm_probe $1 $r 0 0 150; kill $P; summ "$1 nh=$nh raster=$r"
  done
done
done
for nh in 1 2; do VP_NH=$nh timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe dx 16 0 0 1 2>&1 | grep -E "dram|lts|duration" | sed "s/^/nh=$nh dx /"; done
for nh in 1 2; do r=-16; [ $nh = 2 ] && r=-8; VP_NH=$nh timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe dw $r 0 0 1 2>&1 | grep -E "dram|lts|duration" | sed "s/^/nh=$nh dw /"; done

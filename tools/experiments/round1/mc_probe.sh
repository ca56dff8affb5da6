#!/bin/bash
timeout 120 ./tools/gemm_selftest > gpurun_out/selftest_mc.log 2>&1; echo selftest_rc=$?; grep -E "FAIL|SELFTEST" gpurun_out/selftest_mc.log | head -20
sample() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv & echo $!; }
summ() { python - "$1" <<'PY'
import sys, statistics
v=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
v=v[len(v)//4:]
print("   %s: clk median %.0f MHz  power median %.0f W (%d samples)" % (sys.argv[1], statistics.median(float(a) for a,b in v), statistics.median(float(b) for a,b in v), len(v)))
PY
}
for rep in 1 2; do
for k in "k1 0" "dx 16" "dw 0"; do
  set -- $k
  for mc in 1 2; do
    P=$(sample); VP_MC=$mc timeout 120 ./tools/gemm_probe $1 $2 0 0 200; kill $P; summ "$1 mc=$mc"
  done
done
done
for mc in 1 2; do VP_MC=$mc timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe k1 0 0 0 1 2>&1 | grep -E "dram|lts|duration" | sed "s/^/mc=$mc k1 /"; done
for mc in 1 2; do VP_MC=$mc timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe dx 16 0 0 1 2>&1 | grep -E "dram|lts|duration" | sed "s/^/mc=$mc dx /"; done
for mc in 1 2; do VP_MC=$mc timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe dw 0 0 0 1 2>&1 | grep -E "dram|lts|duration" | sed "s/^/mc=$mc dw /"; done

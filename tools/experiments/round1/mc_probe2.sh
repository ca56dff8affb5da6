#!/bin/bash
sample() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv & echo $!; }
summ() { python - "$1" <<'PY'
import sys, statistics
v=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
v=v[len(v)//4:]
print("   %s: clk median %.0f MHz  power median %.0f W (%d samples)" % (sys.argv[1], statistics.median(float(a) for a,b in v), statistics.median(float(b) for a,b in v), len(v)))
PY
}
for rep in 1 2; do
for k in "k1 0" "dx 16" "dx 8" "dw 0"; do
  set -- $k
  for mc in 1 2; do
    P=$(sample); VP_MC=$mc timeout 120 ./tools/gemm_probe $1 $2 0 0 200; kill $P; summ "$1 mc=$mc"
  done
done
done

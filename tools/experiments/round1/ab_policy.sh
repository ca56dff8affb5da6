#!/bin/bash
# interleaved A/B of GEMM L2 policy / raster options inside full bench steps
B="python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for rep in 1 2; do
  for cfg in "" "--opt policy_logits=-1 --opt policy_dx=-1 --opt policy_dw=-1" "--opt raster_dx=8" "--opt raster_logits=16" "--opt policy_dx=-1"; do
    out=$(timeout 200 $B $cfg 2>/dev/null)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-70s %8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
  done
done

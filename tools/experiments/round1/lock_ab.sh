#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
B="python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for rep in 1 2 3; do
  for cfg in "" "--opt lockstep_dx=0 --opt lockstep_dw=0" "--opt lockstep_logits=8"; do
    out=$(timeout 200 $B $cfg 2>/dev/null)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-42s %8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % ('$cfg' or 'default (lockstep dx/dw 8)', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
  done
done

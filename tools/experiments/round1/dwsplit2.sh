#!/bin/bash
B="python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --vocab 32000"
for rep in 1 2; do for cfg in "" "--opt splits_dx=1"; do
  out=$(timeout 200 $B $cfg 2>/dev/null)
  echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-22s %8.0f tok/s %6.3f ms | logits %.3f dx %.3f dw %.3f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
done; done
timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('headline %8.0f tok/s %6.3f ms | logits %.3f dx %.3f dw %.3f | clk %s' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_output_layer.py tests/test_gpu_program.py -m gpu -q -x 2>&1 | tail -2
# an 8-way shard (one rank of N=8): dW split auto vs off
B="python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --vocab 32000"
for rep in 1 2 3; do for cfg in "" "--opt splits_dw=1"; do
  out=$(timeout 200 $B $cfg 2>/dev/null)
  echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-22s %8.0f tok/s %6.3f ms | logits %.3f dx %.3f dw %.3f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
done; done

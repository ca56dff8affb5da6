#!/bin/bash
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|CUDA|error" gpurun_out/selftest.log | head -5
B="python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for rep in 1 2 3; do for cfg in "" "--opt cooperative=0"; do
  out=$(timeout 200 $B $cfg 2>&1 | tail -1)
  echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-22s %8.0f tok/s %6.3f ms | logits %.3f dx %.3f dw %.3f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))" || echo "$out" | tail -3
done; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2

#!/bin/bash
for nh in 2 1; do VP_NH=$nh timeout 120 ./tools/gemm_probe k1 0 0 0 20 | head -3; done
VP_NH=1 timeout 120 ./tools/gemm_probe k1 16 0 0 20 | head -3
for i in 1 2; do for o in "" "--opt nh_logits=1"; do timeout 300 python bench.py --no-cpu-baseline --no-e2e $o > /tmp/b.json 2>/dev/null;
python -c "import json,sys; d=json.load(open('/tmp/b.json')); g=d['roofline']['gemms']; print('%-20s %8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % ('$o' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"; done; done

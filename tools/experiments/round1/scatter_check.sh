#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 120 python bench.py --workload input 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['phase_ms'], d['roofline']['frac'])"; done
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row|k_scatter|k_input" -c 6 python bench.py --workload input --steps 1 --warmup 1 --no-e2e 2>&1 | grep -E "^  [a-z_<>]|duration" | head -12
for i in 1 2; do timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"; done

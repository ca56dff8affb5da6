#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_stats_reduce_ref" -c 2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_stats|duration|dram" | head -6
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q_$i.json 2>/dev/null;
python -c "import json,sys; d=json.load(open('gpurun_out/bench_q_$i.json')); g=d['roofline']['gemms']; print('%8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s | e2e %.0f' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz'], d['e2e']['value']))"; done

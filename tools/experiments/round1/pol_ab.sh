#!/bin/bash
B="python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for rep in 1 2 3; do
  for cfg in "" "--opt policy_logits=-1" "--opt policy_logits=-1 --opt store_evict_first=1"; do
    out=$(timeout 200 $B $cfg 2>/dev/null)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-52s %8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
  done
done
for cfg in "--opt policy_logits=-1" "--opt policy_logits=-1 --opt store_evict_first=1"; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -s 3 -c 1 $B --steps 1 --warmup 1 $cfg 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/ ${cfg} /"
done

#!/bin/bash
# staggered-half MMA schedule (256x512 tiles): GEMM self-test, isolated probes, in-step bench
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest_rc=$?; grep -E "FAIL|SELFTEST" gpurun_out/selftest.log | head -20
for k in "k1 0" "dx 16" "dw -4"; do set -- $k; VP_NH=2 timeout 120 ./tools/gemm_probe $1 $2 0 0 30; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_stagger_$i.json 2>gpurun_out/bench_stagger_$i.err; echo bench_rc=$?;
python -c "import json,sys; d=json.load(open('gpurun_out/bench_stagger_$i.json')); g=d['roofline']['gemms']; print('%8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s | e2e %.0f' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz'], d['e2e']['value']))"; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

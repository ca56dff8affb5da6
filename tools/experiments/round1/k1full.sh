#!/bin/bash
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|CUDA" gpurun_out/selftest.log | head -5
for rep in 1 2; do VP_NH=2 timeout 60 ./tools/gemm_probe k1 0 0 0 30 | grep -E "ideal|issuer|TFLOP"; done
timeout 900 python -m pytest tests/test_gpu_output_layer.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"; done

#!/bin/bash
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|split=" gpurun_out/selftest.log | head -20
for sp in 0 2 3; do VP_NH=2 VP_SPLIT=$sp timeout 120 ./tools/gemm_probe dx 16 0 0 20; done
VP_NH=2 VP_SPLIT=2 timeout 120 ./tools/gemm_probe dx 8 0 0 20
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_split_$i.json 2>gpurun_out/bench_split_$i.err; echo bench_rc=$?;
python -c "import json,sys; d=json.load(open('gpurun_out/bench_split_$i.json')); g=d['roofline']['gemms']; print('%8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % (d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"; done
timeout 900 python -m pytest tests/test_gpu_output_layer.py -m gpu -x -q 2>&1 | tail -3

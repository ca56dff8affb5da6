#!/bin/bash
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|CUDA" gpurun_out/selftest.log | head -5
for rep in 1 2; do for b in gemm_probe gemm_probe_f64; do for k in "dw -4" "dx 16"; do set -- $k; echo "== $b $1"; VP_NH=2 timeout 60 ./tools/$b $1 $2 0 0 30 | grep -E "ideal|issuer|TFLOP"; done; done; done

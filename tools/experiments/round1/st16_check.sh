#!/bin/bash
VP_F32_STORE=2 timeout 300 ./tools/gemm_selftest > gpurun_out/selftest16.log 2>&1; echo selftest16 rc=$?; grep -E "FAIL|SELFTEST|CUDA" gpurun_out/selftest16.log | head -10
for m in 1 2; do for k in "dw -4" "dx 16"; do set -- $k; VP_F32_STORE=$m VP_NH=2 timeout 120 ./tools/gemm_probe $1 $2 0 0 20 | head -2; done; done

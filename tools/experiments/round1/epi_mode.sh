#!/bin/bash
for b in gemm_probe gemm_probe_m3 gemm_probe_m4 gemm_probe_m1; do echo "== $b"; VP_NH=2 timeout 120 ./tools/$b k1 0 0 0 20 | head -2; done
timeout 300 ./tools/vpipe_verify --hidden 4096 --vocab 128256 --devices 8 --batch 1 --seq-len 16; echo verify_rc=$?
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|CUDA" gpurun_out/selftest.log | head -10
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_program.py -m gpu -q 2>&1 | tail -15
timeout 300 ./tools/gemm_selftest > gpurun_out/selftest.log 2>&1; echo selftest rc=$?; grep -E "FAIL|SELFTEST|CUDA" gpurun_out/selftest.log | head -5
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3

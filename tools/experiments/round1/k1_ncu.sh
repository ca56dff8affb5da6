#!/bin/bash
VP_NH=2 timeout 120 ./tools/gemm_probe k1 0 0 0 20
VP_NH=2 timeout 120 ./tools/gemm_probe_poly k1 0 0 0 20
VP_NH=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -s 1 -c 1 -o gpurun_out/k1_epi8 ./tools/gemm_probe k1 0 0 0 1 > gpurun_out/k1_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4

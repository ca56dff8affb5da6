#!/bin/bash
for k in "k1 0" "dx 16" "dw -4"; do set -- $k; VP_NH=2 timeout 120 ./tools/gemm_probe $1 $2 0 0 20; done

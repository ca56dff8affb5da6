#!/bin/bash
for rep in 1 2; do for b in gemm_probe gemm_probe_poly gemm_probe_m1; do echo "== $b"; VP_NH=2 timeout 60 ./tools/$b k1 0 0 0 30 | grep -E "ideal|issuer|TFLOP"; done; done

#!/bin/bash
for p in 8 4 2; do timeout 300 python tools/calibrate.py --p $p --out gpurun_out/calib_p$p.json > /dev/null 2> gpurun_out/calib_p$p.err; echo calib_p$p rc=$?; done

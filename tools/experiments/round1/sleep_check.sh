#!/bin/bash
timeout 120 ./tools/gemm_selftest > gpurun_out/st.log 2>&1; echo selftest_rc=$?; tail -1 gpurun_out/st.log
M="dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum"
for k in "dx 16 2" "dw -4 2"; do set -- $k; VP_NH=$3 timeout 120 ncu --metrics $M --clock-control none -k regex:gemm_sm100 -c 1 ./tools/gemm_probe $1 $2 0 0 1 2>&1 | grep -E "^\s+(dram|lts|gpu__time|sm__cyc|smsp)" | sed "s/^/ours $1 nh=$3 /"; done
./tools/ab3.sh 2>&1 | head -6

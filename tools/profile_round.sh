#!/bin/bash
# Round profile capture (headline config, N=1): bench lines (alg2 headline, alg1, naive, input layer),
# ncu launch list of the bench command, ncu --set full of the three GEMMs and of the input-layer kernels.
# (ncu's kernel replay cannot relaunch cooperative grids: under a profiler the library launches the GEMMs
#  non-cooperatively by itself (NV_NSIGHT_INJECTION_*); --opt cooperative=0 below only makes that explicit.)
R=${1:-r01}
timeout 300 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench_rc=$?
for a in alg1 naive; do timeout 300 python bench.py --alg $a --no-cpu-baseline > gpurun_out/${R}_bench_$a.json 2>/dev/null; echo bench_${a}_rc=$?; done
timeout 300 python bench.py --workload input > gpurun_out/${R}_bench_input.json 2>/dev/null; echo bench_input_rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 3 -c 3 \
  -o gpurun_out/${R}_gemms python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --opt cooperative=0 > gpurun_out/${R}_ncu.log 2>&1; echo ncu_rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_input_forward|k_scatter_rows" -s 6 -c 2 \
  -o gpurun_out/${R}_input python bench.py --workload input --steps 1 --warmup 3 --no-e2e > gpurun_out/${R}_ncu_input.log 2>&1; echo ncu_input_rc=$?

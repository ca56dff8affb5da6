# DRAM bytes per launch (ncu, serialised) of K1 and dW under rasterisation / L2 policy / store-hint combinations
export VP_NH=2 VP_LOCKSTEP=8
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100"
run() { echo "== $*"; timeout 300 ncu $M ./tools/gemm_probe "$@" 1 2>&1 | grep -E "dram__|gpu__time" | awk '{print "   ", $1, $3}'; }
for sef in 0 1; do export VP_SEF=$sef; echo "#### store_evict_first=$sef"
  run k1 16 2 2; run k1 16 2 1; run k1 32 2 1; run k1 24 2 1; run k1 8 2 1
  run dw -4 2 2; run dw -8 2 2; run dw -8 1 2; run dw -4 1 2
  run dx 16 2 2; run dx 32 2 1; run dx 8 2 2
done
timeout 2400 python -m pytest tests/test_gpu_robustness.py -q > gpurun_out/r02n_pytest.log 2>&1; echo pytest_rc=$?
tail -20 gpurun_out/r02n_pytest.log

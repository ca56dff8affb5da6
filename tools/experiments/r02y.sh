# Persisting L2 window (cudaLaunchAttributeAccessPolicyWindow) on the operand re-read across waves:
# DRAM bytes per launch (ncu, serialised) and standalone timing of K1 / dW, vs L2 policies and rasters
export VP_NH=2 VP_LOCKSTEP=8
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -s 1 -c 1 -k regex:gemm_sm100"
run() { echo "== $*  persist=${VP_PERSIST:-0}"; timeout 300 ncu $M ./tools/gemm_probe "$@" 1 2>&1 | grep -E "dram__|gpu__time|lts__|persist|L2 " | awk '{print "   ", $0}'; }
for p in 0 64 96; do export VP_PERSIST=$p
  run dw -4 2 2; run dw -4 0 2; run dw -8 0 2; run dw -8 2 2
done
export VP_SEF=1
for p in 0 40 64 96; do export VP_PERSIST=$p
  run k1 16 2 1; run k1 32 2 1; run k1 32 0 1
done

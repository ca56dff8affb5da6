# fp32-epilogue early release A/B (dx, dw) interleaved; K1 DRAM bytes per raster / policy (ncu, non-cooperative)
export VP_NH=2 VP_LOCKSTEP=8
for rep in 1 2; do
for b in gemm_probe gemm_probe_f32early; do
  echo "== $b dx"; timeout 120 ./tools/$b dx 16 2 2 30 | tail -1
  echo "== $b dw"; timeout 120 ./tools/$b dw -4 2 2 30 | tail -1
done
done
for b in gemm_probe gemm_probe_f32early; do echo "== $b dw probe"; timeout 120 ./tools/$b dw -4 2 2 30 | head -2; done
for r in 16 8 32 4; do
  echo "== ncu k1 raster $r"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100 ./tools/gemm_probe k1 $r 2 2 1 2>&1 | grep -E "dram__|gpu__time|rror"
done
for p in "2 1" "2 0" "0 0" "1 2"; do
  echo "== ncu k1 pol $p"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100 ./tools/gemm_probe k1 16 $p 1 2>&1 | grep -E "dram__|gpu__time"
done
echo "== ncu k1 no lockstep"
VP_LOCKSTEP=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100 ./tools/gemm_probe k1 16 2 2 1 2>&1 | grep -E "dram__|gpu__time"

# K1 early TMEM release A/B (interleaved) + K1 DRAM bytes per rasterisation
export VP_NH=2 VP_LOCKSTEP=8
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader
for rep in 1 2; do
for b in gemm_probe gemm_probe_early gemm_probe_early_poly gemm_probe_poly; do echo "== $b"; timeout 120 ./tools/$b k1 16 2 2 40 | tail -4; done
done
for r in 16 8 32 4; do
  echo "== ncu raster $r"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100 ./tools/gemm_probe_early k1 $r 2 2 1 2>&1 | grep -E "dram__|gpu__time|lts__" 
done
for p in "2 1" "2 0" "0 0"; do
  echo "== ncu pol $p"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1 -c 1 -k regex:gemm_sm100 ./tools/gemm_probe_early k1 16 $p 1 2>&1 | grep -E "dram__|gpu__time"
done

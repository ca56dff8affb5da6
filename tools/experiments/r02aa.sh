# cycle attribution (in-kernel probe, CTA 0) of the three GEMMs at the headline shape, lockstep 8, default rasters/policies
export VP_NH=2 VP_LOCKSTEP=8
for i in 1 2; do
VP_SEF=1 ./tools/gemm_probe k1 16 2 1 20
./tools/gemm_probe dx 16 2 2 20
./tools/gemm_probe dw -4 2 2 20
done

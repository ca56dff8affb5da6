# in-step A/B (interleaved) of the dW GEMM tile shape: 256x512 (default, nh=2) vs 256x256 with double-buffered
# TMEM accumulators (nh_dw=1), with its raster variants
for rep in 1 2 3; do
  for v in default nh1 nh1r8 nh1r2; do
    case $v in default) O="";; nh1) O="--opt nh_dw=1";; nh1r8) O="--opt nh_dw=1 --opt raster_dw=-8";; nh1r2) O="--opt nh_dw=1 --opt raster_dw=-16";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02ai_b.json 2>gpurun_out/r02ai_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02ai_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02ai_b.err
  done
done

# in-step A/B (interleaved): dW rasterisation (N-fastest groups of 4 n-tiles = default, 8 = all n-tiles, 2)
for rep in 1 2 3; do
  for v in r4 r8 r2; do
    case $v in r4) O="";; r8) O="--opt raster_dw=-8";; r2) O="--opt raster_dw=-2";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02at_b.json 2>gpurun_out/r02at_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02at_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02at_b.err
  done
done

# input layer (configs[3]) A/B, interleaved: base vs head (warp-aggregated slot appends in the scatter planning)
for rep in 1 2 3; do
  for ids in uniform zipf; do for v in base head; do
    if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=build_variants/pre_aq/libvpipe_b200.so; fi
    timeout 300 python bench.py --workload input --no-cpu-baseline --no-e2e --steps 50 --ids $ids > gpurun_out/r02bg_b.json 2>gpurun_out/r02bg_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02bg_b.json').read().splitlines()[-1]);r=d['roofline'];print('$v', '$ids', round(d['value']/1e6,2), 'M tok/s', {k:round(v,4) for k,v in r['phase_ms'].items()}, r['kernel'], round(r['frac'],3))" || tail -2 gpurun_out/r02bg_b.err
  done; done
done

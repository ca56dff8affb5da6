# does TMA multicast of B (4-CTA clusters) buy clock under the power cap? NH=1 (256x256 pair tiles) mc=1 vs mc=2, in-step, interleaved
for rep in 1 2; do
  for o in "nh_logits=2 --opt nh_dx=2 --opt nh_dw=2" "nh_logits=1 --opt nh_dx=1 --opt nh_dw=1 --opt multicast=1" "nh_logits=1 --opt nh_dx=1 --opt nh_dw=1 --opt multicast=2"; do
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 --opt $o > gpurun_out/r02s_b.json 2>gpurun_out/r02s_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02s_b.json').read().splitlines()[-1]);print('$o'.replace('--opt ',''), round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -3 gpurun_out/r02s_b.err
  done
done

# in-step A/B (interleaved, one box): K1 with W evict-first + P stores evict-first (DRAM 13.3 -> 9.8 GB per K1 launch)
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 > gpurun_out/r02o_a_$rep.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02o_a_$rep.json').read().splitlines()[-1]);print('default  ', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
  timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 --opt policyb_logits=1 --opt store_evict_first=1 > gpurun_out/r02o_b_$rep.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02o_b_$rep.json').read().splitlines()[-1]);print('pb1+sef1 ', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
  timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 --opt policyb_logits=1 --opt store_evict_first=1 --opt raster_dw=-8 > gpurun_out/r02o_c_$rep.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02o_c_$rep.json').read().splitlines()[-1]);print('+dw-8    ', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
done

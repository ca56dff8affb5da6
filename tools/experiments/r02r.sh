# in-step A/B of the wave-lockstep epoch (k-blocks) per GEMM, interleaved on one box
for rep in 1 2 3; do
  for o in "lockstep_logits=8 --opt lockstep_dx=8 --opt lockstep_dw=8" "lockstep_logits=4 --opt lockstep_dx=4 --opt lockstep_dw=4" "lockstep_logits=2 --opt lockstep_dx=2 --opt lockstep_dw=2" "lockstep_logits=4 --opt lockstep_dx=8 --opt lockstep_dw=4"; do
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 --opt $o > gpurun_out/r02r_b.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02r_b.json').read().splitlines()[-1]);print('$o'.replace('--opt ',''), round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
  done
done

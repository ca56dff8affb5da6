# in-step A/B (interleaved): dW with the persisting window at the default raster (-4), A evict-normal / B evict-last
# (ncu: 8.7 + 4.2 GB per launch), vs default; and the same without the window
for rep in 1 2 3; do
  for v in default pw4 pol02; do
    case $v in default) O="";; pw4) O="--opt persist_dw=1 --opt policy_dw=0 --opt policyb_dw=2";; pol02) O="--opt policy_dw=0 --opt policyb_dw=2";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02ak_b.json 2>gpurun_out/r02ak_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02ak_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02ak_b.err
  done
done

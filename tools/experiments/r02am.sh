# in-step A/B (interleaved): K1 lockstep epoch 2 / 1 with dX and dW at the default 8
for rep in 1 2 3; do
  for v in e8 k1e2 k1e1 k1e2dx4; do
    case $v in e8) O="";; k1e2) O="--opt lockstep_logits=2";; k1e1) O="--opt lockstep_logits=1";;
      k1e2dx4) O="--opt lockstep_logits=2 --opt lockstep_dx=4";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02am_b.json 2>gpurun_out/r02am_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02am_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02am_b.err
  done
done

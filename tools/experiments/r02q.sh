# lockstep epoch sweep for K1 / dW (probe: cycles vs MMA-ideal), then in-step A/B of the best
export VP_NH=2
for ls in 0 4 8 16 32; do
  echo "== k1 lockstep $ls"; VP_LOCKSTEP=$ls timeout 120 ./tools/gemm_probe k1 16 2 1 30 | head -2
done
for ls in 0 8 16; do
  echo "== dw lockstep $ls"; VP_LOCKSTEP=$ls timeout 120 ./tools/gemm_probe dw -4 2 2 30 | head -2
  echo "== dx lockstep $ls"; VP_LOCKSTEP=$ls timeout 120 ./tools/gemm_probe dx 16 2 2 30 | head -2
done
for rep in 1 2; do
  for o in "lockstep_logits=8" "lockstep_logits=0" "lockstep_logits=16"; do
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 --opt $o > gpurun_out/r02q_b.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r02q_b.json').read().splitlines()[-1]);print('$o', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
  done
done

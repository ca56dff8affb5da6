# in-step A/B (interleaved): wave-lockstep epoch (k-blocks) of the three GEMMs: 8 (default) vs 4 vs 2,
# and per-GEMM variants (the standalone probe showed K1's clock rising as the epoch shrinks: r02q)
for rep in 1 2 3; do
  for v in e8 e4 e2 k1e4; do
    case $v in e8) O="";; e4) O="--opt lockstep_logits=4 --opt lockstep_dx=4 --opt lockstep_dw=4";;
      e2) O="--opt lockstep_logits=2 --opt lockstep_dx=2 --opt lockstep_dw=2";; k1e4) O="--opt lockstep_logits=4";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02al_b.json 2>gpurun_out/r02al_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02al_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02al_b.err
  done
done

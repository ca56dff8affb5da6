# in-step A/B (interleaved) of the persisting L2 window: default vs dW (raster -8, A evict-normal, B evict-last,
# X-operand window) vs dW + K1 (raster 32, X window)
DW="--opt persist_dw=1 --opt raster_dw=-8 --opt policy_dw=0 --opt policyb_dw=2"
K1="--opt persist_logits=1 --opt raster_logits=32"
for rep in 1 2 3; do
  for v in default dw dwk1 k1; do
    case $v in default) O="";; dw) O="$DW";; dwk1) O="$DW $K1";; k1) O="$K1";; esac
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 $O > gpurun_out/r02z_b.json 2>gpurun_out/r02z_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02z_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02z_b.err
  done
done

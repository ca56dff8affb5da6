# in-step A/B (interleaved): round-2 HEAD before this session (0dc4455, build_variants/base) vs the current build
for rep in 1 2 3; do
  for v in base head; do
    if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=build_variants/$v/libvpipe_b200.so; fi
    timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --steps 20 > gpurun_out/r02ac_b.json 2>gpurun_out/r02ac_b.err
    python -c "import json;d=json.loads(open('gpurun_out/r02ac_b.json').read().splitlines()[-1]);print('$v', round(d['value']), d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})" || tail -2 gpurun_out/r02ac_b.err
  done
done

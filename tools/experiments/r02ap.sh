# A/B (interleaved): batched loads in k_stats_reduce_ref; configs[0] (graph replay and eager) and the headline
export VPIPE_LIB_BASE=build_variants/pre_ap/libvpipe_b200.so
for rep in 1 2 3; do
  for v in base head; do
    if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=$VPIPE_LIB_BASE; fi
    timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/r02ap_c0.json 2>/dev/null
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-graph --steps 20 > gpurun_out/r02ap_h.json 2>/dev/null
    python -c "
import json
c=json.loads(open('gpurun_out/r02ap_c0.json').read().splitlines()[-1]); h=json.loads(open('gpurun_out/r02ap_h.json').read().splitlines()[-1])
print('$v', 'c0', round(c['value']/1e6,3), 'graph', round(c['graph']['value']/1e6,3), 'headline', round(h['value']), h['clocks']['sm_mhz'])"
  done
done

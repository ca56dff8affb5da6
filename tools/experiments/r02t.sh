# input layer: persistent scatter-apply (warp per unique row) + unrolled gather
timeout 900 python -m pytest tests/test_gpu_input_layer.py tests/test_gpu_loopback.py tests/test_gpu_extensions.py -q -x > gpurun_out/r02t_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r02t_pytest.log
for ids in uniform zipf; do for rep in 1 2; do
  timeout 300 python bench.py --workload input --ids $ids --no-cpu-baseline > gpurun_out/r02t_in_$ids.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02t_in_$ids.json').read().splitlines()[-1]);print('$ids', round(d['value']), d['ms_per_step'], d['roofline'].get('phase_ms'), d['e2e']['value'])"
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_input_forward|k_sc_" -s 12 -c 6 python bench.py --workload input --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_input|k_sc|dram__|gpu__time|warps_active" | head -40

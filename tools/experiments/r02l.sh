# new GPU tests (extensions, robustness) + memory-bounded alg2 at a long-context shape
timeout 2400 python -m pytest tests/test_gpu_extensions.py tests/test_gpu_robustness.py -x -q --durations=10 > gpurun_out/r02l_pytest.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/r02l_pytest.log
for c in 0 16384 8192 4096; do
  timeout 600 python bench.py --tokens 65536 --steps 5 --warmup 3 --no-graph --no-cpu-baseline --chunk-tokens $c > gpurun_out/r02l_long_c$c.json 2>gpurun_out/r02l_long_c$c.err; echo rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/r02l_long_c$c.json').read().splitlines()[-1]);print('chunk', $c, d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['config'].get('P_bytes'), {k:round(v['tflops'],1) for k,v in d['roofline']['gemms'].items()})"
done

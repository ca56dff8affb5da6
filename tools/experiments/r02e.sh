timeout 600 python -m pytest tests/test_gpu_input_layer.py tests/test_gpu_loopback.py -x -q -k "input" > gpurun_out/r02e_input.log 2>&1; echo input_rc=$?
tail -30 gpurun_out/r02e_input.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r02e_pytest.log
for ids in uniform zipf; do timeout 300 python bench.py --workload input --ids $ids --no-cpu-baseline --no-e2e > gpurun_out/r02e_input_$ids.json 2>&1; echo bench_$ids=$?; python -c "
import json; d=json.loads(open('gpurun_out/r02e_input_$ids.json').read().splitlines()[-1]); r=d['roofline']; print('$ids', d['value'], d['ms_per_step'], r['phase_ms'], r['achieved'], r['frac'], d['config']['distinct_rows'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sc_|k_input" --csv python bench.py --workload input --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_uniform.csv 2>&1; echo ncu=$?
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sc_|k_input" --csv python bench.py --workload input --ids zipf --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_zipf.csv 2>&1; echo ncu=$?
grep -E "k_sc|k_input" gpurun_out/r02e_ncu_uniform.csv | tail -24
grep -E "k_sc|k_input" gpurun_out/r02e_ncu_zipf.csv | tail -24

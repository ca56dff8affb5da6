timeout 600 python -m pytest tests/test_gpu_input_layer.py -x -q > gpurun_out/r02g_input.log 2>&1; echo input_rc=$?
tail -3 gpurun_out/r02g_input.log
for ids in uniform zipf; do timeout 300 python bench.py --workload input --ids $ids --no-cpu-baseline --no-e2e > gpurun_out/r02g_input_$ids.json 2>&1; echo bench_$ids=$?; python -c "
import json; d=json.loads(open('gpurun_out/r02g_input_$ids.json').read().splitlines()[-1]); r=d['roofline']; print('$ids', d['value'], d['ms_per_step'], r['phase_ms'], r['achieved'], r['frac'], d['config']['distinct_rows'])"; done
for ids in uniform zipf; do timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sc_apply" --csv python bench.py --workload input --ids $ids --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02g_ncu_$ids.csv 2>&1; echo ncu=$?
grep -E "k_sc" gpurun_out/r02g_ncu_$ids.csv | tail -3 | awk -F'","' '{print $(NF-2), $NF}'; done

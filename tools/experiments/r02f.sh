timeout 600 python -m pytest tests/test_gpu_input_layer.py -x -q > gpurun_out/r02f_input.log 2>&1; echo input_rc=$?
tail -3 gpurun_out/r02f_input.log
for ids in uniform zipf; do timeout 300 python bench.py --workload input --ids $ids --no-cpu-baseline --no-e2e > gpurun_out/r02f_input_$ids.json 2>&1; echo bench_$ids=$?; python -c "
import json; d=json.loads(open('gpurun_out/r02f_input_$ids.json').read().splitlines()[-1]); r=d['roofline']; print('$ids', d['value'], d['ms_per_step'], r['phase_ms'], r['achieved'], r['frac'], d['config']['distinct_rows'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sc_apply" --csv python bench.py --workload input --ids zipf --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02f_ncu_zipf.csv 2>&1; echo ncu=$?
grep -E "k_sc" gpurun_out/r02f_ncu_zipf.csv | tail -3
for b in gemm_probe gemm_probe_m3 gemm_probe_m4 gemm_probe_m1 gemm_probe_m2; do echo "== $b"; VP_NH=2 VP_LOCKSTEP=8 timeout 120 ./tools/$b k1 16 2 2 20 | head -4; done

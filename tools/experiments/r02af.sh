# final profile of the round-2 build (fused exchange): bench lines (headline, reference arm, alg1, naive,
# input uniform/zipf, configs 0-2), launch list, ncu --set full of the GEMMs and the input kernels
R=r02af
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2>/dev/null; echo ref_rc=$?
for a in alg1 naive; do timeout 300 python bench.py --alg $a --no-cpu-baseline > gpurun_out/${R}_bench_$a.json 2>/dev/null; echo bench_${a}_rc=$?; done
timeout 300 python bench.py --workload input > gpurun_out/${R}_bench_input.json 2>/dev/null; echo input_rc=$?
timeout 300 python bench.py --workload input --ids zipf --no-cpu-baseline > gpurun_out/${R}_bench_input_zipf.json 2>/dev/null; echo zipf_rc=$?
timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline > gpurun_out/${R}_c0.json 2>/dev/null; echo c0_rc=$?
timeout 300 python bench.py --vocab 128256 --no-cpu-baseline > gpurun_out/${R}_llama.json 2>/dev/null; echo llama_rc=$?
timeout 300 python bench.py --tokens 4096 --hidden 3584 --vocab 32000 --no-cpu-baseline > gpurun_out/${R}_gemma_shard8.json 2>/dev/null; echo gemma_rc=$?
python - <<'PY'
import json
for f in ["bench", "bench_ref", "bench_alg1", "bench_naive", "bench_input", "bench_input_zipf", "c0", "llama", "gemma_shard8"]:
    try:
        d = json.loads(open(f"gpurun_out/r02af_{f}.json").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f, round(d["value"]), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"),
              r.get("frac"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 3 -c 3 \
  -o gpurun_out/${R}_gemms python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${R}_ncu.log 2>&1; echo ncu_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_input_forward|k_sc_" -s 12 -c 6 \
  -o gpurun_out/${R}_input python bench.py --workload input --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_input.log 2>&1; echo ncu_input_rc=$?
ls -la gpurun_out/ | grep $R
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --dry-run --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_dry2.json 2>/dev/null; echo dry2_rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --workload input --gpus 4 --dry-run --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_dry4_input.json 2>/dev/null; echo dry4_input_rc=$?

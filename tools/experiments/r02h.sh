# round-2 session 2: re-validate HEAD on a B200 (GPU tests, headline bench, 2-rank dry run, launch list)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02h_pytest.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/r02h_pytest.log
timeout 300 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo bench_rc=$?
cat gpurun_out/r02h_bench.json
timeout 300 python bench.py --impl reference > gpurun_out/r02h_bench_ref.json 2>&1; echo ref_rc=$?; tail -1 gpurun_out/r02h_bench_ref.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --dry-run --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_dry2.json 2> gpurun_out/r02h_dry2.err; echo dry2_rc=$?; tail -2 gpurun_out/r02h_dry2.json; tail -5 gpurun_out/r02h_dry2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r02h_launches.log 2>&1; echo launches_rc=$?
grep -c '"' gpurun_out/r02h_launches.csv; grep -i error gpurun_out/r02h_launches.csv gpurun_out/r02h_launches.log | head

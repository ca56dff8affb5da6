set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
make -C paper_2411_05288_b200/csrc -q || echo "lib stale?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; echo bench_rc=$?; cat gpurun_out/bench_$i.json; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref_rc=$?; cat gpurun_out/bench_ref.json

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02a_pytest.log
timeout 300 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench_rc=$?
cat gpurun_out/r02a_bench.json | head -c 3000

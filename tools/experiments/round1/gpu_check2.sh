set -x
timeout 900 python -m pytest tests/test_gpu_output_layer.py -m gpu -x -q -k "widths or memcheck" > gpurun_out/pytest_new.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_new.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
bash tools/profile_round.sh r01b

# loopback (nranks > 1 on one GPU) tests, then the whole GPU suite
export VPIPE_LOOPBACK_TIMEOUT=90
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -v > gpurun_out/r02b_loopback.log 2>&1; echo loopback_rc=$?
tail -40 gpurun_out/r02b_loopback.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_loopback.py > gpurun_out/r02b_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/r02b_pytest.log

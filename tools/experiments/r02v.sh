timeout 1200 python -m pytest tests/test_gpu_extensions.py tests/test_gpu_loopback.py -q -x --durations=5 > gpurun_out/r02v_pytest.log 2>&1; echo pytest_rc=$?; tail -12 gpurun_out/r02v_pytest.log

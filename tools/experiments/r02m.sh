# extensions + robustness + loopback (owner gather) GPU tests
timeout 2400 python -m pytest tests/test_gpu_extensions.py tests/test_gpu_robustness.py tests/test_gpu_loopback.py -q --durations=12 > gpurun_out/r02m_pytest.log 2>&1; echo pytest_rc=$?
tail -45 gpurun_out/r02m_pytest.log

export VPIPE_LOOPBACK_TIMEOUT=90
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_cpp_api.py -x -q --durations=0 > gpurun_out/r02c_loopback.log 2>&1; echo loopback_rc=$?
tail -40 gpurun_out/r02c_loopback.log
timeout 300 python -m pytest tests/test_gpu_output_layer.py -x -q -k "logit_shift or Y_and_B" > gpurun_out/r02c_new.log 2>&1; echo new_rc=$?
tail -30 gpurun_out/r02c_new.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_loopback.py > gpurun_out/r02c_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/r02c_pytest.log

# The S >= 8 C1 parity tests and every conv launch configuration, then the whole gpu suite.
set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_c1_sessions.py tests/test_gpu_conv_configs.py -q -s --timeout 600 -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1
tail -40 gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider --deselect tests/test_gpu_c1_sessions.py --deselect tests/test_gpu_conv_configs.py > gpurun_out/pytest.log 2>&1
tail -5 gpurun_out/pytest.log

set -x
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x --timeout 120 -p no:cacheprovider -k "conv" > gpurun_out/pytest_conv.log 2>&1
tail -30 gpurun_out/pytest_conv.log

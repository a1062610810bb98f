set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
tail -5 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-budget 10 > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log

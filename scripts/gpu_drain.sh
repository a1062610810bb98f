set -x
TAG=default timeout 300 python scripts/diag_c1_sessions.py 32 32 2>&1 | grep -E '^\[|Error|error' | head -5
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none 2>&1 | tail -1 | cut -c1-300
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_drain2.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/launch_diff.py gpurun_out/l_nodrain.csv gpurun_out/l_drain2.csv
timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_conv_configs.py tests/test_gpu_c1_sessions.py -q -s --timeout 300 -p no:cacheprovider > gpurun_out/pytest_d4.log 2>&1
tail -8 gpurun_out/pytest_d4.log

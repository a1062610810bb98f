set -x
for S in 1 8 32; do TAG=default timeout 180 python scripts/diag_c1_sessions.py $S 8 2>&1 | grep '^\[' ; done
TAG=drain1 EVC_DRAIN=1 timeout 180 python scripts/diag_c1_sessions.py 32 8 2>&1 | grep '^\['
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none 2>&1 | tail -1 | cut -c1-400
EVC_DRAIN=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none 2>&1 | tail -1 | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_conv_configs.py tests/test_gpu_graph.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3

set -x
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -k conv -p no:cacheprovider 2>&1 | tail -3
python scripts/conv_bench.py --mode incr --trace 2>&1 | grep -v "start spread" | tee gpurun_out/convbench_trace.txt

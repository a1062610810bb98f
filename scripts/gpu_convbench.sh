timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python scripts/conv_bench.py --mode incr --trace --layers dec3,dec2 2>&1 | tee gpurun_out/convbench_trace.txt
python scripts/step_breakdown.py --sessions 1 > gpurun_out/brk_s1.txt 2>&1
python scripts/step_breakdown.py --sessions 32 > gpurun_out/brk_s32.txt 2>&1

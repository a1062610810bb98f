python scripts/conv_bench.py --mode incr --trace --layers dec3,dec2,res0a 2>&1 | tee gpurun_out/convbench_trace.txt

timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 2>&1 | tail -4
timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0,res0a,enc1 --iters 20 2>&1 | tee gpurun_out/convbench.txt
timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0,res0a,enc1 --sessions 32 --iters 5 2>&1 | tee gpurun_out/convbench32.txt
timeout 300 python scripts/step_breakdown.py --sessions 1 > gpurun_out/brk_s1.txt 2>&1
timeout 300 python scripts/step_breakdown.py --sessions 32 > gpurun_out/brk_s32.txt 2>&1

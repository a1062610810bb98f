timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_conv_fused" -s 3 -c 1 -o gpurun_out/prof_dec2 python scripts/conv_bench.py --mode incr --layers dec2 --iters 1 > gpurun_out/ncu_dec2.log 2>&1
tail -1 gpurun_out/ncu_dec2.log

export EVC_SUBPIXEL=1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_subpix_border" --launch-skip 1 -c 1 -o gpurun_out/subk python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_subk.log 2>&1
python scripts/ncu_summary.py gpurun_out/subk.ncu-rep > gpurun_out/subk.txt 2>&1; cat gpurun_out/subk.txt
python scripts/cuda_hot.py gpurun_out/subk.ncu-rep 30 > gpurun_out/subk_hot.txt 2>&1; cat gpurun_out/subk_hot.txt

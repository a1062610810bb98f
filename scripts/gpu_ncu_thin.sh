# full ncu capture of the enc0 thin conv (first k_conv_thin launch of a step) at S=32
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_thin" -s 0 -c 1 -o gpurun_out/prof_thin_s32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_thin.log 2>&1
tail -1 gpurun_out/ncu_thin.log

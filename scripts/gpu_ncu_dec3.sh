# full ncu capture of the dec3 conv launch (15th conv-family launch of a step) at S=32
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv" -s 14 -c 1 -o gpurun_out/prof_dec3_s32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_dec3.log 2>&1
tail -1 gpurun_out/ncu_dec3.log

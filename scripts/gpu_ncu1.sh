timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_fused" -s 10 -c 1 -o gpurun_out/prof_conv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_f.log 2>&1
tail -1 gpurun_out/ncu_f.log
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_fused" -s 10 -c 1 -o gpurun_out/prof_conv_s32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_f32.log 2>&1
tail -1 gpurun_out/ncu_f32.log

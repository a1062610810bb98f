# dominant conv launch (dec3, persistent BN=16) at 32 streams: full set; and the DRAM bytes of every conv launch of one step
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_persist<16>" -c 1 -o gpurun_out/prof_dec3_s32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_f32.log 2>&1
tail -1 gpurun_out/ncu_f32.log
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_conv" --csv --log-file gpurun_out/conv_traffic_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_t32.log 2>&1
tail -1 gpurun_out/ncu_t32.log

timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_up_sparsify" -s 3 -c 1 -o gpurun_out/prof_ups32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_ups.log 2>&1
tail -1 gpurun_out/ncu_ups.log

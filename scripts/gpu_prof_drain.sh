set -x
EVC_DRAIN=0 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_nodrain.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_drain.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/launch_diff.py gpurun_out/l_nodrain.csv gpurun_out/l_drain.csv

timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launch.csv python scripts/profile_c2.py > gpurun_out/c2p.log 2>&1
cat gpurun_out/c2p.log | grep -v "^==" ; python scripts/launch_diff.py gpurun_out/c2_launch.csv gpurun_out/c2_launch.csv 2>/dev/null | awk '{print $1, $2, $3, $(NF-2)}' | head -60
for sc in enc0 enc0,enc1 enc1; do timeout 300 python scripts/profile_c2.py --scatter $sc 2>&1 | grep "C2 S"; done

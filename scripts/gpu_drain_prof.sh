for D in 1000 4; do
  EVC_DRAIN=$D timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_conv --csv --log-file gpurun_out/lf_$D.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
done

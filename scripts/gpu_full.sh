# Full ncu captures of selected launches (indices into one profiled C1 step): bash scripts/gpu_full.sh 35 11 31
set -x
for L in "$@"; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -s $L -c 1 -o gpurun_out/full_$L python scripts/profile_step.py --steps 1 > gpurun_out/ncu_full_$L.log 2>&1
tail -1 gpurun_out/ncu_full_$L.log
done

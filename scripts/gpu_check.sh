set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
tail -15 gpurun_out/pytest.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --steps 2 > gpurun_out/prof.log 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1.csv --steps 2 | head -30
timeout 600 python bench.py --steps 64 --warmup 3 --cpu-budget 10 > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log

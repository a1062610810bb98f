# Iteration pass: gpu tests, C1 launch list, short bench, conv microbench.
set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
tail -25 gpurun_out/pytest.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --steps 2 > gpurun_out/prof.log 2>&1
tail -3 gpurun_out/prof.log
python scripts/kernel_summary.py gpurun_out/launches_c1.csv --steps 2 > gpurun_out/kernel_summary.txt; head -30 gpurun_out/kernel_summary.txt
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
python scripts/conv_bench.py --mode incr --trace > gpurun_out/convbench_trace.txt 2>&1; tail -40 gpurun_out/convbench_trace.txt

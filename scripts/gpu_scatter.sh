timeout 300 python -m pytest tests/test_gpu_scatter.py -q -x -s --timeout 120 -p no:cacheprovider > gpurun_out/pytest_sc.log 2>&1; tail -30 gpurun_out/pytest_sc.log
timeout 300 python scripts/c4_bench.py > gpurun_out/c4.log 2>&1; head -12 gpurun_out/c4.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sc_launch.csv python scripts/scatter_prof.py > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/sc_launch.csv | head -14

# One GPU pass: smoke, gpu tests, launch list, bench (with CPU baseline), full ncu of the top conv launch.
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
tail -5 gpurun_out/pytest.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --steps 2 > gpurun_out/prof.log 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1.csv --steps 2 > gpurun_out/kernel_summary.txt; head -20 gpurun_out/kernel_summary.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/prof32.log 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1_s32.csv --steps 1 > gpurun_out/kernel_summary_s32.txt; head -20 gpurun_out/kernel_summary_s32.txt
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_conv" --csv --log-file gpurun_out/conv_traffic_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_t32.log 2>&1
python scripts/conv_traffic.py gpurun_out/conv_traffic_s32.csv --sessions 32 > gpurun_out/conv_traffic_s32.json; head -4 gpurun_out/conv_traffic_s32.json
cp gpurun_out/conv_traffic_s32.json profiles/r01_conv_traffic_s32.json
timeout 900 python bench.py --steps 64 --warmup 3 --cpu-budget 15 > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 8 --warmup 3 --cpu-budget 20 > gpurun_out/bench_ref.log 2>&1; tail -2 gpurun_out/bench_ref.log
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv" -s 14 -c 1 -o gpurun_out/prof_conv python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_f.log 2>&1
tail -1 gpurun_out/ncu_f.log
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_up_sparsify" -s 3 -c 1 -o gpurun_out/prof_ups32 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_ups.log 2>&1

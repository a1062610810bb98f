# Per-kernel key metrics for every launch of one C1 step + full captures of selected kernels.
set -x
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_membar,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg"
timeout 900 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/ncu_metrics.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_m.log 2>&1
tail -2 gpurun_out/ncu_m.log
# warm-cache variant (no L2 flush between kernels), closer to graph replay
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_warm.csv python scripts/profile_step.py --steps 2 > gpurun_out/ncu_w.log 2>&1
python scripts/kernel_summary.py gpurun_out/launches_warm.csv --steps 2 | head -20
# full captures: res conv (launch 30), res sparsify k_tiles<1,4> (28), dec3 up_sparsify (87)
for L in 27 30 87; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -s $L -c 1 -o gpurun_out/full_$L python scripts/profile_step.py --steps 1 > gpurun_out/ncu_full_$L.log 2>&1
tail -1 gpurun_out/ncu_full_$L.log
done

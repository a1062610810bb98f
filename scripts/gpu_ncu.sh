set -x
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__occupancy_limit_shared_mem,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_short_scoreboard,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__average_warp_latency_issue_stalled_lg_throttle,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"
timeout 900 ncu --profile-from-start off --clock-control none --metrics $M -k regex:"k_tiles|k_conv_tma|k_conv_flags|k_conv_count|k_upsample|k_region_reduce" --csv --log-file gpurun_out/ncu_metrics.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_m.log 2>&1
tail -2 gpurun_out/ncu_m.log
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_tma" -s 14 -c 1 -o gpurun_out/prof_conv_dec3 python scripts/profile_step.py --steps 1 > gpurun_out/ncu_f.log 2>&1
tail -2 gpurun_out/ncu_f.log
ls -la gpurun_out

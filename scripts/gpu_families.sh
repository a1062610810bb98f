# ncu evidence for every kernel family (profiles/r02_*): one launch list with DRAM bytes, then
# --set full captures of one instance of each family's kernel
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/fam_launch.csv python scripts/profile_families.py > gpurun_out/fam.log 2>&1
tail -2 gpurun_out/fam.log
for k in k_diff_mask k_sparsify_small k_conv_thin k_tiles k_up_sparsify k_conv_persist k_conv_fused k_integrate_flat k_meter_step k_to_hwc k_compact_write k_event_runs k_count_scatter k_ingest_ring k_encode_windows; do
  c=1; [ "$k" = "k_tiles" ] && c=3
  timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"$k" -c $c -o gpurun_out/fam_$k python scripts/profile_families.py > /dev/null 2>&1
  echo "$k rc=$?"
done
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_scatter|k_scatter_gather" -c 2 -o gpurun_out/fam_scatter python scripts/scatter_prof.py > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | wc -l

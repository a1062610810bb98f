# ncu evidence for every kernel family (profiles/r02_*): one launch list with DRAM bytes, then
# --set full captures of one instance of each family's kernel
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/fam_launch.csv python scripts/profile_families.py > gpurun_out/fam.log 2>&1
tail -2 gpurun_out/fam.log
for k in k_diff_mask k_sparsify_small k_conv_thin k_tiles k_up_sparsify k_subpix_input k_subpix_border k_conv_persist k_conv_fused k_integrate_flat k_meter_step k_to_hwc k_compact_write k_event_runs k_count_scatter k_ingest_ring k_encode_windows; do
  c=1; [ "$k" = "k_tiles" ] && c=3
  timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"$k" -c $c -o gpurun_out/fam_$k python scripts/profile_families.py > /dev/null 2>&1
  echo "$k rc=$?"
done
# the sub-pixel dec3 conv (third persistent launch of the step) and its input pass (second)
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_persist --launch-skip 2 -c 1 -o gpurun_out/fam_z_dec3_subpixel_conv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_subpix_input --launch-skip 1 -c 1 -o gpurun_out/fam_z_dec3_subpix_input python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_scatter|k_scatter_gather" -c 2 -o gpurun_out/fam_scatter python scripts/scatter_prof.py > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | wc -l
timeout 300 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_conv" --csv --log-file gpurun_out/conv_traffic_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/conv_traffic.py gpurun_out/conv_traffic_s32.csv --sessions 32 > gpurun_out/r02_conv_traffic_s32.json; head -5 gpurun_out/r02_conv_traffic_s32.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1
python scripts/families_summary.py gpurun_out > gpurun_out/r02_ncu_families.md 2> gpurun_out/fam_sum.err
for f in gpurun_out/fam_*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>/dev/null; done
ls -la gpurun_out/*.ncu-rep | awk '{s+=$5} END {print s/1e6, "MB of reports"}'
# keep the dec3 sub-pixel conv and input-pass reports for source-level reading; drop the rest
mkdir -p gpurun_out/keep; mv gpurun_out/fam_z_dec3_subpixel_conv.ncu-rep gpurun_out/fam_z_dec3_subpix_input.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep; du -sh gpurun_out
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_noSub_s32.csv env EVC_SUBPIXEL=0 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1_s32.csv > gpurun_out/r02_kernel_summary_s32.txt 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1.csv --steps 2 > gpurun_out/r02_kernel_summary.txt 2>&1
python scripts/kernel_summary.py gpurun_out/launches_c1_noSub_s32.csv > gpurun_out/r02_kernel_summary_s32_highres_decoder.txt 2>&1
cat gpurun_out/fam_*.txt > gpurun_out/r02_ncu_family_summaries.txt

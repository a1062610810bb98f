# border GEMM: input channels split across warp halves for C_out <= 16; min 4 (default) vs 3 CTAs/SM
timeout 900 python -m pytest tests/test_gpu_subpixel.py tests/test_gpu_c1_sessions.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -3
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main sb3; do
  if [ $v = sb3 ]; then cp paper_2303_04670_b200/libevconv_sb3.so paper_2303_04670_b200/libevconv.so; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b_$v.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
  echo "== $v"; python scripts/kernel_summary.py gpurun_out/launches_b_$v.csv --steps 1 > gpurun_out/ks_b_$v.txt; grep -i "launches\|subpix" gpurun_out/ks_b_$v.txt
done
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so

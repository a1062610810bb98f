# --set full of the dec3 conv at 32 streams: high-res (packed persist<16>) vs sub-pixel (composed persist<64>)
EVC_NO_SUBPIXEL=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_persist<16" -c 1 -o gpurun_out/dec3_hi python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_hi.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_conv_persist" --launch-skip 2 -c 1 -o gpurun_out/dec3_sub python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_sub.log 2>&1
for r in dec3_hi dec3_sub; do
  python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1
  python scripts/sass_hot.py gpurun_out/$r.ncu-rep 40 > gpurun_out/${r}_hot.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda > gpurun_out/${r}_src.csv 2>gpurun_out/${r}_src.err
done
ls -la gpurun_out/dec3_*

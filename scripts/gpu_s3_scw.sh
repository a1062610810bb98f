# warp-wide MMA issue in the scatter conv (C4): parity + sweep vs the lane-0 issuer
timeout 600 python -m pytest tests/test_gpu_scatter.py tests/test_gpu_c4.py -q -x -p no:cacheprovider 2>&1 | tail -2
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main sclane0; do
  if [ $v = sclane0 ]; then cp paper_2303_04670_b200/libevconv_sclane0.so paper_2303_04670_b200/libevconv.so; else cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so; fi
  echo "== $v"; timeout 300 python scripts/c4_bench.py > gpurun_out/c4_$v.log 2>&1; head -9 gpurun_out/c4_$v.log
done
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so

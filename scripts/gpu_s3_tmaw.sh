# warp-wide TMA producer (elected lane issues each TMA / bulk copy / expect_tx) vs the lane-0 producer
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main tmaw; do
  if [ $v = tmaw ]; then cp paper_2303_04670_b200/libevconv_tmaw.so paper_2303_04670_b200/libevconv.so; else cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so; fi
  echo "== $v"; timeout 300 python scripts/conv_bench.py --mode incr --layers enc1,enc2,res0a,dec0,dec1 --sessions 32 --iters 10 2>&1 | grep -v trace | tail -6
  timeout 300 python scripts/conv_bench.py --mode incr --layers dec2,dec3 --subpixel --sessions 32 --iters 10 2>&1 | tail -3
done
cp paper_2303_04670_b200/libevconv_tmaw.so paper_2303_04670_b200/libevconv.so
timeout 900 python -m pytest tests/test_gpu_conv_configs.py tests/test_gpu_c1_sessions.py tests/test_gpu_subpixel.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -3
timeout 600 python bench.py --steps 32 > gpurun_out/bench_tmaw.json 2> gpurun_out/bench_tmaw.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_tmaw.json').read().strip().splitlines()[-1])
print('tmaw value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50',round(d['p50_ms'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'e2e',round(d['e2e']['value']), 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],3))
"
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so

# warp-wide MMA issue (elect.sync inside the asm, no per-MMA waterfall loop) vs the lane-0 issuer
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main mmaw main; do
  if [ $v = mmaw ]; then cp paper_2303_04670_b200/libevconv_mmaw.so paper_2303_04670_b200/libevconv.so; else cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so; fi
  echo "== $v"; timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,enc3,res0a,dec0 --sessions 32 --iters 10 2>&1 | tail -5
done
cp paper_2303_04670_b200/libevconv_mmaw.so paper_2303_04670_b200/libevconv.so
timeout 900 python -m pytest tests/test_gpu_conv_configs.py tests/test_gpu_c1_sessions.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -3
timeout 600 python bench.py --steps 32 > gpurun_out/bench_mmaw.json 2> gpurun_out/bench_mmaw.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_mmaw.json').read().strip().splitlines()[-1])
print('mmaw value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50',round(d['p50_ms'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'e2e',round(d['e2e']['value']), 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],3))
"
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so

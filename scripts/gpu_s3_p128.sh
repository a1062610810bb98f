# persistent BN = 128 (split-small TMEM) A/B + thin-conv launch-bound variants + parity of the touched paths
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
echo "== persist128 (default)"; timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,enc3,res0a,dec0 --sessions 32 --iters 10 2>&1 | tee gpurun_out/p128_on.txt
echo "== one-shot"; EVC_NO_PERSIST128=1 timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,enc3,res0a,dec0 --sessions 32 --iters 10 2>&1 | tee gpurun_out/p128_off.txt
echo "== dense persist128"; timeout 300 python scripts/conv_bench.py --mode dense --layers enc2,dec0 --sessions 32 --iters 10 2>&1 | tail -3
echo "== enc0 thin default"; timeout 120 python scripts/conv_bench.py --mode incr --layers enc0,pred3 --sessions 32 --iters 10 2>&1 | tail -3
for v in thin4 thin4s6; do cp paper_2303_04670_b200/libevconv_$v.so paper_2303_04670_b200/libevconv.so; echo "== enc0 $v"; timeout 120 python scripts/conv_bench.py --mode incr --layers enc0,pred3 --sessions 32 --iters 10 2>&1 | tail -3; done
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so
timeout 900 python -m pytest tests/test_gpu_c1_sessions.py tests/test_gpu_conv_configs.py tests/test_gpu_parity_configs.py tests/test_gpu_subpixel.py -x -q -p no:cacheprovider -s 2>&1 | tail -25 > gpurun_out/p128_tests.log; tail -5 gpurun_out/p128_tests.log
timeout 900 python bench.py --steps 32 > gpurun_out/bench_p128.json 2> gpurun_out/bench_p128.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_p128.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_p128.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3), 'frac', d['roofline']['frac'])
"

# dec1 / sub-pixel dec3 (C_out <= 64, row mode, 2 pipeline stages) vs tap mode / BN 32 at 32 streams
for env in "" "EVC_NO_ROW=1" "EVC_FORCE_BN=32" "EVC_NO_ROW=1 EVC_FORCE_BN=32"; do
  echo "== [$env] dec1"; env $env timeout 120 python scripts/conv_bench.py --mode incr --layers dec1,enc1 --sessions 32 --iters 10 2>&1 | grep -v trace | tail -3
  echo "== [$env] dec3 sub-pixel"; env $env timeout 120 python scripts/conv_bench.py --mode incr --layers dec3,dec2 --subpixel --sessions 32 --iters 10 2>&1 | tail -3
done
timeout 600 python -m pytest tests/test_gpu_conv_configs.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --steps 32 > gpurun_out/bench_rt.json 2> gpurun_out/bench_rt.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_rt.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_rt.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3), 'frac', d['roofline']['frac'])
"

# session-3 re-entry check: driver-style GPU tests, default bench, conv phase traces at 32 streams
start=$(date +%s)
timeout 1200 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_driver.log 2>&1; echo "pytest rc=$? $(( $(date +%s) - start )) s"
tail -3 gpurun_out/pytest_driver.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3), 'frac', d['roofline']['frac'])
"
timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,res0a,dec0,dec1 --sessions 32 --iters 5 --trace 2>&1 | tee gpurun_out/convtrace32.txt

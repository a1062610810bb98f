# final evidence of the round: driver-style GPU tests, smoke, default bench, reference arm
start=$(date +%s)
timeout 1800 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_driver.log 2>&1; echo "pytest rc=$? $(( $(date +%s) - start )) s"
tail -3 gpurun_out/pytest_driver.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_final.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),d['e2e']['run_values'],'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3), 'frac', d['roofline']['frac'], 'clocks', d['clocks'])
for k,v in d.get('configs',{}).items(): print(k, {kk: v[kk] for kk in ('value','p50_increment_latency_ms') if kk in v} if isinstance(v,dict) else v)
"
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; tail -1 gpurun_out/bench_reference.json | cut -c1-300

# warp-wide MMA issue in both conv kernels (default) vs the lane-0 issuer: persistent layers, full GPU suite, bench
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main lane0; do
  if [ $v = lane0 ]; then cp paper_2303_04670_b200/libevconv_lane0.so paper_2303_04670_b200/libevconv.so; else cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so; fi
  echo "== $v"; timeout 300 python scripts/conv_bench.py --mode incr --layers enc1,dec1 --sessions 32 --iters 10 2>&1 | tail -3
  timeout 300 python scripts/conv_bench.py --mode incr --layers dec2,dec3 --subpixel --sessions 32 --iters 10 2>&1 | tail -3
done
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so
start=$(date +%s)
timeout 1800 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_driver.log 2>&1; echo "pytest rc=$? $(( $(date +%s) - start )) s"
tail -2 gpurun_out/pytest_driver.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mmaw.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_mmaw.csv --steps 1 > gpurun_out/ks_mmaw.txt; head -10 gpurun_out/ks_mmaw.txt
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50',round(d['p50_ms'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),d['e2e']['run_values'],'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3),'frac',d['roofline']['frac'],'clocks',d['clocks'])
for k,v in d.get('configs',{}).items(): print(k, {kk: v[kk] for kk in ('value','p50_increment_latency_ms') if kk in v} if isinstance(v,dict) else v)
"

# L2 prefetch of the activation accumulators by the epilogue warps (EVC_NO_ACC_PREFETCH=1 = off)
for v in on off; do
  if [ $v = off ]; then export EVC_NO_ACC_PREFETCH=1; else unset EVC_NO_ACC_PREFETCH; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pf_$v.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
  echo "== $v"; python scripts/kernel_summary.py gpurun_out/launches_pf_$v.csv --steps 1 > gpurun_out/ks_pf_$v.txt; head -9 gpurun_out/ks_pf_$v.txt
  timeout 600 python bench.py --steps 32 > gpurun_out/bench_pf_$v.json 2> gpurun_out/bench_pf_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/bench_pf_$v.json').read().strip().splitlines()[-1])
print('$v value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']), 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],3))
"
done
unset EVC_NO_ACC_PREFETCH
timeout 900 python -m pytest tests/test_gpu_conv_configs.py tests/test_gpu_c1_sessions.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|S=8\|passed\|failed" | tail -4

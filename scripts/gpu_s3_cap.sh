# dense graph captured right after the first eager dense pass (no capture inside timed runs) + up_sparsify mask trim
timeout 1500 python -m pytest tests/test_gpu_refresh_graph.py tests/test_gpu_serving.py tests/test_gpu_ingest.py tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_ops.py tests/test_gpu_parity_configs.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -4
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cap.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_cap.csv --steps 1 > gpurun_out/ks_cap.txt; head -8 gpurun_out/ks_cap.txt
for r in 1 2; do
timeout 600 python bench.py > gpurun_out/bench_cap$r.json 2> gpurun_out/bench_cap$r.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cap$r.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50',round(d['p50_ms'],3),'p99',round(d['p99_ms'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']), d['e2e']['run_values'])
"
done

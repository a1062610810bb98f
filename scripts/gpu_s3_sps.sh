# input sparsify skipping dead tiles: parity (graph tests incl. C1 at 8 / 32 streams, C2, C3, serving) + launch list + bench
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_parity_configs.py tests/test_gpu_serving.py tests/test_gpu_ingest.py tests/test_gpu_determinism.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -5
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sps.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_sps.csv --steps 1 > gpurun_out/ks_sps.txt; cat gpurun_out/ks_sps.txt
timeout 600 python bench.py > gpurun_out/bench_sps.json 2> gpurun_out/bench_sps.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_sps.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']), d['e2e']['run_values'], 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],3))
"

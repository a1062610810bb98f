# trimmed upsample loop in the sub-pixel input pass: parity + launch list + bench
timeout 900 python -m pytest tests/test_gpu_subpixel.py tests/test_gpu_c1_sessions.py tests/test_gpu_ops.py tests/test_gpu_graph.py -x -q -p no:cacheprovider -s 2>&1 | grep -i "S=32\|passed\|failed\|Error" | tail -4
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sub2.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_sub2.csv --steps 1 > gpurun_out/ks_sub2.txt; head -8 gpurun_out/ks_sub2.txt
timeout 600 python bench.py > gpurun_out/bench_sub2.json 2> gpurun_out/bench_sub2.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_sub2.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']), d['e2e']['run_values'], 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],3))
"

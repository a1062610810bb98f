timeout 1500 python -m pytest tests/test_gpu_conv_configs.py tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_subpixel.py tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -3
summ() { python -c "
import json;d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1 value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),d['e2e'].get('run_values'),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3))"; }
timeout 600 python bench.py --steps 10 --warmup 3 --configs none > gpurun_out/bench_b.json 2> /dev/null; summ gpurun_out/bench_b.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sub_s32.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/launches_sub_s32.csv 2>&1 | head -12

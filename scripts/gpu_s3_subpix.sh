# hoisted-row sub-pixel input pass: parity (bit-exact flags, values) + per-kernel launch list at 32 streams + bench
timeout 900 python -m pytest tests/test_gpu_subpixel.py tests/test_gpu_c1_sessions.py tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -3
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s32.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/kernel_summary.py gpurun_out/launches_s32.csv --steps 1 | tee gpurun_out/kernel_summary_s32.txt
timeout 900 python bench.py > gpurun_out/bench_sp.json 2> gpurun_out/bench_sp.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_sp.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_sp.json').read().strip().splitlines()[-1])
print('value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3), 'frac', d['roofline']['frac'])
"

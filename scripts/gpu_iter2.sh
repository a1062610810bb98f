timeout 900 python -m pytest tests/test_gpu_subpixel.py tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_conv_configs.py -x -q -p no:cacheprovider 2>&1 | tail -3
summ() { python -c "
import json;d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1 value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']),'gemm_ms',round(d['roofline']['gemm_ms_per_step'],3))"; }
timeout 600 python bench.py --steps 10 --warmup 3 --configs none > gpurun_out/bench_it.json 2> gpurun_out/bench_it.err; summ gpurun_out/bench_it.json
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_up_sparsify --launch-skip 3 -c 1 -o gpurun_out/up_dec3 python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_up.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_persist --launch-skip 3 -c 1 -o gpurun_out/dec3_hi python scripts/profile_step.py --steps 1 --sessions 32 > gpurun_out/ncu_hi.log 2>&1
for r in up_dec3 dec3_hi; do
  python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; cat gpurun_out/$r.txt
  python scripts/cuda_hot.py gpurun_out/$r.ncu-rep 40 > gpurun_out/${r}_hot.txt 2>&1
done

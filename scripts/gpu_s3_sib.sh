# fused sub-pixel input pass + border GEMM (one launch) vs the two launches; ingest one step ahead (serving)
timeout 900 python -m pytest tests/test_gpu_subpixel.py tests/test_gpu_serving.py tests/test_gpu_ingest.py -x -q -p no:cacheprovider 2>&1 | tail -3
cp paper_2303_04670_b200/libevconv.so /tmp/libevconv_main.so
for v in main split sib3; do
  if [ $v = sib3 ]; then cp paper_2303_04670_b200/libevconv_sib3.so paper_2303_04670_b200/libevconv.so; fi
  if [ $v = split ]; then export EVC_SUBPIX_SPLIT=1; else unset EVC_SUBPIX_SPLIT; fi
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv timeout 600 python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
  echo "== $v"; python scripts/kernel_summary.py gpurun_out/launches_$v.csv --steps 1 | head -9
  timeout 600 python bench.py --steps 32 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1])
print('$v value',round(d['value']),'ms',round(d['ms_per_step'],3),'p50 s1',round(d['p50_increment_latency_ms'],3),'refresh',round(d['refresh_ms'],2),'e2e',round(d['e2e']['value']), d['e2e'].get('run_values'))
"
done
cp /tmp/libevconv_main.so paper_2303_04670_b200/libevconv.so

for S in 1 32; do
  timeout 600 python bench.py --steps 32 --warmup 3 --sessions $S --no-cpu-baseline --no-latency-pass > gpurun_out/bench_S$S.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_S$S.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('S=$S', d and (round(d['value'],1), round(d['p50_ms'],3), d['e2e']['value'], d['roofline']['achieved'], d['roofline']['gemm_ms_per_step']))
" || tail -5 gpurun_out/bench_S$S.log
done

for P in 1 0; do
EVC_PDL=$P timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$P.log 2>&1
python -c "
import json
d=json.loads([x for x in open('gpurun_out/bench_pdl$P.log') if x.startswith('{')][-1])
print('PDL=$P', round(d['value'],1), round(d['p50_ms'],4), d['e2e']['value'])"
done

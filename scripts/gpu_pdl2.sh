for p in 0 1; do
  echo "== EVC_PDL=$p"
  EVC_PDL=$p timeout 200 python bench.py --steps 32 --warmup 3 --sessions 1 --no-cpu-baseline --configs none > gpurun_out/b_pdl.json 2>&1
  python - <<'P'
import json; d=json.loads(open('gpurun_out/b_pdl.json').read().strip().splitlines()[-1]); print('S=1', {k: d[k] for k in ('value','p50_ms','p99_ms')})
P
  EVC_PDL=$p timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/b_pdl.json 2>&1
  python - <<'P'
import json; d=json.loads(open('gpurun_out/b_pdl.json').read().strip().splitlines()[-1]); print('S=32', {k: d[k] for k in ('value','p50_ms')})
P
done

for D in 1 2 4; do
  echo "== EVC_DRAIN=$D"
  EVC_DRAIN=$D TAG=d$D timeout 300 python scripts/diag_c1_sessions.py 32 32 2>&1 | grep -E '^\[|Error|error' | head -5
  EVC_DRAIN=$D timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/bench_dd.json 2>&1
  python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_dd.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','value_no_refresh','refresh_ms','p50_ms')})
P
done

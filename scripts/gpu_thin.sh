for v in 8 16; do
  echo "== EVC_THIN_COUT=$v"
  EVC_THIN_COUT=$v TAG=thin$v timeout 300 python scripts/diag_c1_sessions.py 32 16 2>&1 | grep -E '^\[' | head -5
  EVC_THIN_COUT=$v timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/bench_thin.json 2>&1
  python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_thin.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','value_no_refresh','refresh_ms','p50_ms')})
P
  EVC_THIN_COUT=$v timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_$v.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
  python scripts/kernel_summary.py gpurun_out/lt_$v.csv | head -10
done

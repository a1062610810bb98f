timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_determinism.py tests/test_gpu_serving.py tests/test_gpu_recurrent.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3
TAG=denseup timeout 300 python scripts/diag_c1_sessions.py 32 16 2>&1 | grep -E '^\[' | head -5
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/bench_du.json 2>&1
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_du.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','value_no_refresh','refresh_ms','p50_ms')}, d['e2e']['value'])
P

for t in $(python -m pytest tests/test_gpu_conv_configs.py --collect-only -q 2>/dev/null | grep "::" | grep chain); do
  timeout 90 python -m pytest "$t" -q -x -p no:cacheprovider > /tmp/t.log 2>&1; rc=$?; [ $rc -ne 0 ] && echo "FAIL rc=$rc $t $(tail -3 /tmp/t.log | head -1)"
done
echo chain-configs-done
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py tests/test_gpu_determinism.py tests/test_gpu_serving.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3
TAG=fuse timeout 300 python scripts/diag_c1_sessions.py 32 16 2>&1 | grep -E '^\[' | head -5
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/bench_df.json 2>&1
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_df.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','value_no_refresh','refresh_ms','p50_ms')}, d['e2e']['value'])
P

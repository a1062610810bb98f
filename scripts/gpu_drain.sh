timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_conv --csv --log-file gpurun_out/lf_new.csv python scripts/profile_step.py --steps 1 --sessions 32 > /dev/null 2>&1
python scripts/kernel_summary.py gpurun_out/lf_new.csv | head -9
TAG=default timeout 300 python scripts/diag_c1_sessions.py 32 32 2>&1 | grep -E '^\[|Error|error' | head -5
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs none > gpurun_out/bench_d6.json 2>&1; tail -1 gpurun_out/bench_d6.json | cut -c1-200
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_d6.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','value_no_refresh','refresh_ms','p50_ms','ms_per_step')})
P
for t in $(python -m pytest tests/test_gpu_conv_configs.py --collect-only -q 2>/dev/null | grep "::"); do
  timeout 90 python -m pytest "$t" -q -x -p no:cacheprovider > /tmp/t.log 2>&1; rc=$?; [ $rc -ne 0 ] && echo "FAIL rc=$rc $t $(tail -3 /tmp/t.log | head -1)"
done
echo conv-configs-done
timeout 600 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_c1_sessions.py tests/test_gpu_recurrent.py tests/test_gpu_replay.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_d6.log 2>&1; tail -3 gpurun_out/pytest_d6.log

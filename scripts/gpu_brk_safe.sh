# gpu tests + step breakdowns, each under its own timeout (new synchronisation code)
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_brk.log 2>&1; tail -2 gpurun_out/pytest_brk.log
timeout 120 python scripts/step_breakdown.py --sessions 1 > gpurun_out/brk_s1.txt 2>&1
timeout 120 python scripts/step_breakdown.py --sessions 32 > gpurun_out/brk_s32.txt 2>&1

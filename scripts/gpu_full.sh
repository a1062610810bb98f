# full GPU pass: smoke, every gpu test (conv configs one process each), bench with sub-configs
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for t in $(python -m pytest tests/test_gpu_conv_configs.py --collect-only -q 2>/dev/null | grep "::"); do
  timeout 90 python -m pytest "$t" -q -x -p no:cacheprovider > /tmp/t.log 2>&1; rc=$?; [ $rc -ne 0 ] && echo "FAIL rc=$rc $t $(tail -3 /tmp/t.log | head -1)"
done
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_conv_configs.py > gpurun_out/pytest_full.log 2>&1; tail -4 gpurun_out/pytest_full.log
grep "^PARITY\|^S=\|ConvLSTM\|recurrent UNet" gpurun_out/pytest_full.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 3000 gpurun_out/bench_full.json

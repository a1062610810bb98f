# exactly the driver's round-end commands (one pytest process for every gpu test), then the default bench
start=$(date +%s)
timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_driver.log 2>&1; echo "pytest rc=$? $(( $(date +%s) - start )) s"
tail -3 gpurun_out/pytest_driver.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$? $(( $(date +%s) - start )) s"
tail -3 gpurun_out/r02_bench.err

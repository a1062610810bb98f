# sub-pixel decoder convs: parity first, then the C1 graph tests and a quick bench
timeout 600 python -m pytest tests/test_gpu_subpixel.py -x -q -s -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_c1_sessions.py -x -q -p no:cacheprovider 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 --configs none > gpurun_out/bench_sub.json 2> gpurun_out/bench_sub.err; tail -c 1500 gpurun_out/bench_sub.json; tail -3 gpurun_out/bench_sub.err

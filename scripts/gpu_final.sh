start=$(date +%s)
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$? $(( $(date +%s) - start )) s"
start=$(date +%s)
timeout 900 python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$? $(( $(date +%s) - start )) s"
tail -c 600 gpurun_out/r02_bench_reference.json
EVC_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --sessions 8 --configs none --no-cpu-baseline --no-latency-pass > gpurun_out/r02_bench_2rank_shared.json 2> gpurun_out/r02_2rank.err; echo "2rank rc=$?"
tail -c 400 gpurun_out/r02_bench_2rank_shared.json; tail -3 gpurun_out/r02_2rank.err

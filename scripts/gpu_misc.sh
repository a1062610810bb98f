export PYTHONFAULTHANDLER=1
for r in 0 1; do
  EVC_BENCH_SHARE_GPU=1 RANK=$r LOCAL_RANK=$r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 \
    timeout -s ABRT 240 python bench.py --gpus 2 --steps 5 --warmup 3 --sessions 8 --configs none --no-cpu-baseline \
    --no-latency-pass > gpurun_out/r2_$r.out 2> gpurun_out/r2_$r.err &
done
wait
tail -c 500 gpurun_out/r2_0.out; echo
EVC_BENCH_SHARE_GPU=1 timeout -s ABRT 300 python bench.py --gpus 2 --steps 5 --warmup 3 --sessions 8 --configs none --no-cpu-baseline --no-latency-pass > gpurun_out/r02_bench_2rank_shared.json 2> gpurun_out/r2t.err; echo "torchrun rc=$?"; tail -c 300 gpurun_out/r02_bench_2rank_shared.json; echo
timeout 300 python scripts/two_streams.py 32 2
timeout 300 python scripts/two_streams.py 32 4

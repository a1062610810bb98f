# N > 1 bench logic on a one-GPU box (EVC_BENCH_SHARE_GPU=1: both ranks on GPU 0 over gloo), two attempts
export PYTHONFAULTHANDLER=1
for ifn in "" lo; do
  echo "== GLOO_SOCKET_IFNAME=$ifn"
  for r in 0 1; do
    GLOO_SOCKET_IFNAME=$ifn EVC_BENCH_SHARE_GPU=1 RANK=$r LOCAL_RANK=$r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 \
      timeout -s ABRT 150 python bench.py --gpus 2 --steps 5 --warmup 3 --sessions 8 --configs none --no-cpu-baseline \
      --no-latency-pass > gpurun_out/r2_$r.out 2> gpurun_out/r2_$r.err &
  done
  wait
  tail -c 300 gpurun_out/r2_0.out; echo; grep -A 12 "most recent call first" gpurun_out/r2_0.err | head -30; tail -3 gpurun_out/r2_1.err
  [ -s gpurun_out/r2_0.out ] && break
done
timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-latency-pass --configs c4 > gpurun_out/bench_c4.json 2>&1; tail -c 300 gpurun_out/bench_c4.json

for env in "" "EVC_DRAIN=6" "EVC_DRAIN=8"; do
  echo "== [$env]"; env $env timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,res0a,dec0,dec1 --sessions 32 --iters 10 2>&1 | grep -v trace | tail -5
done

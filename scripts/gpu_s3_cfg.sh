# conv configuration re-check after the warp-wide MMA issue (32 streams, warm)
for env in "" "EVC_FORCE_SPLITS=2" "EVC_FORCE_BN=64" "EVC_FORCE_RW=16"; do
  echo "== [$env]"; env $env timeout 300 python scripts/conv_bench.py --mode incr --layers enc2,enc3,res0a,dec0 --sessions 32 --iters 10 2>&1 | grep -v trace | tail -5
done
for env in "" "EVC_FORCE_SPLITS=2" "EVC_FORCE_BN=64"; do
  echo "== [$env] dec2 sub-pixel"; env $env timeout 300 python scripts/conv_bench.py --mode incr --layers dec2 --subpixel --sessions 32 --iters 10 2>&1 | tail -2
done

L=enc2,enc3,res0a,dec0
for env in "" "EVC_FORCE_SPLITS=2" "EVC_FORCE_SPLITS=3" "EVC_FORCE_BN=64" "EVC_DRAIN=8" "EVC_DRAIN=16"; do
  echo "== $env"
  env $env timeout 200 python scripts/conv_bench.py --sessions 32 --layers $L --iters 30 2>&1 | grep -v "^$" | tail -5
done

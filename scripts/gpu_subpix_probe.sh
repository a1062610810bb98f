# what-if probe: decoder convs as sub-pixel convs on the low-res input (4x output channels), forced configs
S=32; it=5
timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0 --sessions $S --iters $it 2>&1 | tail -5
timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0 --sessions $S --iters $it --subpixel 2>&1 | tail -5
for bn in 16 32 64 128; do
  EVC_FORCE_BN=$bn timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0 --sessions $S --iters $it --subpixel 2>&1 | tail -5
done
EVC_NO_ROW=1 timeout 300 python scripts/conv_bench.py --mode incr --layers dec3,dec2,dec1,dec0 --sessions $S --iters $it --subpixel 2>&1 | tail -5

# A/B build: recompile one source with extra nvcc flags and link libevconv_<name>.so next to the default
# library (the GPU script copies it over libevconv.so to time it).
#   bash scripts/build_variant.sh <name> <source.cu> "<nvcc flags>"
set -e
name=$1; src=$2; extra=$3
P=paper_2303_04670_b200; B=$P/build; V=$B/variant_$name; mkdir -p $V
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -Xptxas -warn-spills -I include $extra -c $P/csrc/$src -o $V/${src%.cu}.o
objs=""; for o in $B/*.o; do b=$(basename $o); if [ -f $V/$b ]; then objs="$objs $V/$b"; else objs="$objs $o"; fi; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $P/libevconv_$name.so $objs
echo built $P/libevconv_$name.so

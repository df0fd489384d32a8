#!/usr/bin/env bash
# Build an A/B variant of libprefillonly.so with extra -D flags on one source file:
#   tools/build_variant.sh NAME SOURCE "-DFOO=1 -DBAR=0"   ->  build/variants/lib_NAME.so
# Run a tool against it with PREFILLONLY_LIB=build/variants/lib_NAME.so.
set -euo pipefail
name=$1; src=$2; flags=${3:-}
cd "$(dirname "$0")/.."
make -s -j8 >/dev/null
out=build/variants/$name; mkdir -p "$out"
base=$(basename "$src" .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -Iinclude -Xptxas -v $flags -c "paper_2505_07203_b200/csrc/$src" -o "$out/$base.o" \
  2> "$out/$base.ptxas.txt" || { cat "$out/$base.ptxas.txt"; exit 1; }
objs=$(ls build/obj/*.o | grep -v "/$base.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "build/variants/lib_$name.so" $objs \
  "$out/$base.o" -lcuda -L/usr/local/cuda/lib64/stubs
grep -E "Used [0-9]+ registers|spill" "$out/$base.ptxas.txt" | grep -B1 -A0 "attn_fwd" >/dev/null || true
echo "build/variants/lib_$name.so"

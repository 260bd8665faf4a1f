#!/bin/sh
# Build an A/B variant of the library with extra nvcc flags:
#   tools/build_variant.sh NAME -DFLAG=VALUE ...  ->  paper_1705_07175_b200/lib/libbitnn_b200_NAME.so
# (load it with B2_LIB=<path> for an experiment; the package default stays libbitnn_b200.so)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_1705_07175_b200/lib/libbitnn_b200_$name.so
tmp=$(mktemp -d)
for f in paper_1705_07175_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -Iinclude "$@" -c "$f" -o "$tmp/$(basename "$f").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o "$out" "$tmp"/*.o -lcudart_static
rm -rf "$tmp"
echo "$out"

#!/bin/bash
# Build a variant library with extra -D knobs for one source file:
#   tools/build_variant.sh NAME SRC "-DJ2D_RING=8 ..."  -> build/var/NAME/libtvstencil.so
# (select it at run time with TVSTENCIL_LIB=build/var/NAME/libtvstencil.so)
set -e
name=$1; src=$2; defs=$3
cd "$(dirname "$0")/.."
make -s -j16 >/dev/null
mkdir -p build/var/$name
objs=""
for o in build/*.o; do
  b=$(basename $o .o)
  if [ "$b" = "$src" ]; then
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $defs \
      -c -o build/var/$name/$b.o paper_2010_04868_b200/csrc/$b.cu
    objs="$objs build/var/$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$name/libtvstencil.so $objs
echo built build/var/$name/libtvstencil.so

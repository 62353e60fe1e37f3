#!/bin/bash
# Builds paper_1412_1885_b200/lib/libtenkit_b200_<name>.so: the library with ttm_stream.cu recompiled
# under extra -D flags (compile-time A/B of the stream kernel); select it with TENKIT_B200_LIB=<path>.
# usage: tools/build_variant.sh <name> -DTK_STREAM_NA_MAX=2 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
pkg=$root/paper_1412_1885_b200
python -c "import sys; sys.path.insert(0, '$root'); from paper_1412_1885_b200 import build_ext; build_ext.build()"
obj=$pkg/build/ttm_stream_$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$root/include "$@" \
  -c $pkg/csrc/ttm_stream.cu -o $obj
objs=$(ls $pkg/build/*.o | grep -v "ttm_stream" | tr '\n' ' ')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $pkg/lib/libtenkit_b200_$name.so $objs $obj
echo built $pkg/lib/libtenkit_b200_$name.so

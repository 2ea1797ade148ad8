#!/bin/bash
# Build a variant of the library with extra nvcc flags into lib/<name>.so,
# reusing the main build's objects except the streaming-evaluator units.
# usage: scripts/build_variant.sh NAME "-DXE_FOO=1 ..." [object glob to rebuild, default eval_stream*]
set -e
cd "$(dirname "$0")/../paper_2212_09290_b200/csrc"
make -j16 >/dev/null
rm -rf ../../build/obj_$1 && cp -rp ../../build/obj ../../build/obj_$1
rm -f ../../build/obj_$1/${3:-eval_stream*}.o
make -j16 BUILD=../../build/obj_$1 OUT=../lib/$1.so XFLAGS="$2" >/dev/null
echo built ../lib/$1.so

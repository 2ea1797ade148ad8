#!/bin/bash
# K2b A/B over library builds (XE_LIB): config-5 placements/s of each
for lib in "$@"; do
  echo "== $lib"
  XE_LIB_LENIENT=1 XE_LIB=$PWD/$lib timeout 300 python scripts/place_ab.py 4000000 2>&1 | grep sliced=1
done

#!/bin/bash
# A/B a configuration over alternative builds of libstc.so: tools/ab_lib.sh <config> lib1.so lib2.so ...
cfg=$1; shift
for lib in "$@"; do
  cp "$lib" paper_2405_16883_b200/libstc.so
  echo "== $lib"; timeout 300 python tools/bench_configs.py --configs "$cfg" 2>&1 | tail -1 | cut -c1-100
done

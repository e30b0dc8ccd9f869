#!/bin/bash
# A/B a configuration over library builds, interleaved rounds: tools/ab.sh <cfg> <rounds> lib1.so lib2.so ...
cfg=$1; rounds=$2; shift 2
for r in $(seq 1 $rounds); do
  for lib in "$@"; do STC_LIBRARY=$PWD/$lib timeout 300 python tools/ab_time.py $cfg 2>&1 | tail -1; done
done

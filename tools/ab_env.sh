#!/usr/bin/env bash
# single-problem latency with and without an environment switch:  bash tools/ab_env.sh VAR=value
O=gpurun_out/abenv; mkdir -p $O
for rep in 1 2 3; do
  echo -n "base: " >> $O/out.txt; timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
  echo -n "$1: " >> $O/out.txt; env "$1" timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
done

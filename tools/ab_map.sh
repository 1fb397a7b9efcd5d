#!/usr/bin/env bash
# single-problem latency: mapped-result publication vs D2H copy-back (PRRTC_NO_MAP=1)
O=gpurun_out/abmap; mkdir -p $O
for rep in 1 2 3; do
  echo -n "map:  " >> $O/out.txt; timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
  echo -n "copy: " >> $O/out.txt; PRRTC_NO_MAP=1 timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
done

#!/usr/bin/env bash
# chunk-latency profile of two library builds: bash tools/ab_chunk.sh libA libB
for lib in "$@"; do
  for r in panda fetch baxter; do
    echo "== $lib $r"; PRRTC_B200_LIB=$lib python tools/chunk_profile.py $r 2>&1 | tail -3
  done
done

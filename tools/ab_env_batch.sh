#!/usr/bin/env bash
# batch throughput with and without an environment switch:  bash tools/ab_env_batch.sh VAR=value
O=gpurun_out/abenvb; mkdir -p $O
for rep in 1 2; do
  echo -n "base: " >> $O/out.txt; timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-extras --latency-samples 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']), d['success_rate'])" >> $O/out.txt
  echo -n "$1: " >> $O/out.txt; env "$1" timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-extras --latency-samples 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']), d['success_rate'])" >> $O/out.txt
done

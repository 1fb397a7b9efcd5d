#!/usr/bin/env bash
# A/B an environment knob on the bench headline (device-resident value and e2e),
# alternating runs in one box session:  bash tools/ab_knob.sh VAR "a b" [reps] [robot]
VAR=$1; VALS=$2; REPS=${3:-3}; ROBOT=${4:-panda}
for r in $(seq $REPS); do
  for v in $VALS; do
    env $VAR=$v python bench.py --robot $ROBOT --steps 20 --no-extras --no-parity --no-cpu-baseline --latency-samples ${LAT:-30} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v', round(d['value']), round(d['e2e']['value']), round(d['success_rate'],3), round(d['latency_ms']['median'],4), round(d['latency_ms']['p95'],4))"
  done
done

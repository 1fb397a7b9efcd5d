T=$1
mkdir -p gpurun_out/$T
for i in 1 2 3; do timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-extras --latency-samples 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['e2e']['value']), d['latency_ms']['median'], d['success_rate'])"; done > gpurun_out/$T/bq.txt

#!/usr/bin/env bash
# one iteration of the GPU loop: parity suite, chunk phases, bench line (no
# CPU baseline), batch work split. Output under gpurun_out/<tag>/.
T=${1:-it}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in panda fetch baxter; do timeout 100 python tools/chunk_profile.py $r >> $O/chunk.txt 2>&1; done
timeout 400 python bench.py --steps 10 --no-cpu-baseline --latency-samples 100 > $O/bench.json 2> $O/bench.err
for r in panda baxter; do timeout 200 python tools/batch_work.py $r > $O/work_$r.txt 2>&1; done

#!/bin/bash
# C3 lookup-hit-ratio sweep: one bench line per h, into gpurun_out/c3_sweep.jsonl
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
O=gpurun_out
mkdir -p $O
: > $O/c3_sweep.jsonl
for h in 0 0.1 0.2 0.3 0.4 0.5 0.6 0.7 0.8 0.9; do
  timeout 600 python bench.py --config c3 --hit-ratio $h --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline >> $O/c3_sweep.jsonl 2>> $O/c3_sweep.err
done

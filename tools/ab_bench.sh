#!/bin/bash
# A/B(/C...) of prebuilt library variants (ab/*.so) on one box, interleaved:
# bash tools/ab_bench.sh [rounds] [bench args...]   -> gpurun_out/ab.jsonl
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O
R=${1:-3}; shift
: > $O/ab.jsonl
for i in $(seq $R); do
  for f in ab/*.so; do
    v=$(basename $f .so)
    cp $f paper_2604_17353_b200/_lib/liblcb200.so
    LCB_NO_BUILD=1 timeout 600 python bench.py --no-cpu-baseline --no-check "$@" 2>/dev/null | sed "s/^{/{\"variant\": \"$v\", /" >> $O/ab.jsonl
  done
done

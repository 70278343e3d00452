#!/bin/bash
# Wave engine: GPU tests (reference-engine traces, eager and graph), throughput with the decode loop
# eager / replayed from the per-shape graph cache, and the launch list of one eager wave.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_engine.py -q > $O/pytest_engine.log 2>&1; echo "rc=$?" >> $O/pytest_engine.log
for gm in 0; do
 for sh in "256 128" "1024 64"; do set -- $sh
  LCB_ENGINE_GRAPH=$gm timeout 300 python tools/bench_engine.py --requests $1 --tokens $2 > $O/eng_g${gm}_$1x$2.json 2>&1
 done
done
LCB_ENGINE_GRAPH=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/eng_launches.csv python tools/bench_engine.py --requests 256 --tokens 128 --waves 1 > $O/eng_ncu.log 2>&1

#!/bin/bash
# Small-batch checks: adaptive producer grab size (stage / wide kernels), engine decode graph.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kept.py tests/test_gpu_engine.py -q -x > $O/pytest_sb.log 2>&1; echo "rc=$?" >> $O/pytest_sb.log
timeout 600 python bench.py --no-cpu-baseline > $O/sb_c2.json 2> $O/sb_c2.err
for G in 8 4 2; do
  timeout 600 python bench.py --config c5 --one-rank-of $G --no-cpu-baseline > $O/sb_c5_g$G.json 2> $O/sb_c5_g$G.err
done
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/sb_c3.json 2> $O/sb_c3.err
for gm in 1 0; do
 for sh in "256 128" "1024 64"; do set -- $sh
  LCB_ENGINE_GRAPH=$gm timeout 300 python tools/bench_engine.py --requests $1 --tokens $2 > $O/sb_eng_g${gm}_$1x$2.json 2>&1
 done
done
timeout 900 python bench.py --config c4 --cpu-seconds 5 > $O/sb_c4.json 2> $O/sb_c4.err

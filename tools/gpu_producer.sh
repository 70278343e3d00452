#!/bin/bash
# Producer change: fill tests vs the oracle, the engine traces, the C3 miss path (h = 0) and the engine.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_cache_fixes.py -q -x > $O/pytest_prod.log 2>&1; echo "rc=$?" >> $O/pytest_prod.log
timeout 600 python bench.py --config c3 --hit-ratio 0 --steps 5 --warmup 3 --no-cpu-baseline > $O/c3_h0.json 2> $O/c3_h0.err
for sh in "256 128" "1024 64"; do set -- $sh
  timeout 300 python tools/bench_engine.py --requests $1 --tokens $2 > $O/eng_$1x$2.json 2>&1
done

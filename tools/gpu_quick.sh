#!/bin/bash
# quick GPU iteration: gpu tests + c2 bench (no CPU baseline) + resample profile counters
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python tools/prof_resample.py --V 32000 --rows 16384 --draws 32 --top-p 0.9 --bf16 --iters 3 > $O/prof.log 2>&1

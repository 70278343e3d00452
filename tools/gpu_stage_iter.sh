#!/bin/bash
# stage-kernel iteration: parity tests of the staged path, phase profile at the C2 shape, C2 bench (no CPU arm)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "staged or kept or resample_matches or golden" > $O/pytest_stage.log 2>&1; echo "rc=$?" >> $O/pytest_stage.log
LCB_STAGE_PROF=1 timeout 300 python tools/prof_resample.py --V 32000 --rows 16384 --draws 32 --top-p 0.9 --bf16 --iters 3 > $O/prof_c2.log 2>&1
timeout 300 python tools/prof_resample.py --V 32000 --rows 16384 --draws 32 --top-p 0.9 --bf16 --iters 3 --conc 0.0 > $O/prof_c2_flat.log 2>&1
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > $O/bench_c2.json 2> $O/bench_c2.err

#!/bin/bash
# One GPU round: gpu tests, smoke, every bench line (C2 default + reference arm, C1, C3, C5, C4,
# C2 windowed replay, C3 hit-ratio sweep, hotspot replay), the C2 ncu launch list and full captures
# of the hot kernels AT THEIR BENCH LAUNCHES (C2 stage_kernel, C1 rowwarp_kernel, C3 wide_kernel).
set -x
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in c1 c3 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --policy windowed --no-cpu-baseline > $O/bench_c2w.json 2> $O/bench_c2w.err
timeout 900 python bench.py --config c4 --cpu-seconds 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c1 --policy hotspot --no-cpu-baseline > $O/bench_c1h.json 2> $O/bench_c1h.err
STEPS=5 bash tools/c3_sweep.sh
LCB_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-check > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 8 -c 1 -o $O/stage -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-check > $O/ncu_stage.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowwarp_kernel -s 8 -c 1 -o $O/rowwarp -f \
    python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-check > $O/ncu_rowwarp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_kernel -s 5 -c 1 -o $O/wide -f \
    python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-check > $O/ncu_wide.log 2>&1
echo done

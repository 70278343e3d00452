#!/bin/bash
# compute-sanitizer over GPU tests that launch every kernel family (staged K1s, wide K1w,
# row-warp / CTA / exact tiers, probs, cache insert/lookup/pin, replay, hotspots, engine).
# Logs -> gpurun_out/sanitize_<tool>.log ("ERROR SUMMARY: 0 errors" per process = clean).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
FILES="tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_kept.py tests/test_gpu_hotspots.py tests/test_gpu_cache_fixes.py"
ALL="resample_golden_cases or forced_tiers or staged_kernel_edge_rows or wide_kernel_matches_oracle_and_cta_kernel or probs_api_golden or cache_replays_reference_traces or cache_warp_policy_stress or replay_stepwise or replay_hotspot or miss_path or hotspots_golden or engine or writeback or kept_sets_golden or kept_greedy or cache_fixes or narrow"
SMALL="resample_golden_cases or staged_kernel_edge_rows or (wide_kernel_matches_oracle_and_cta_kernel and 151936-0.0) or cache_replays_reference_traces or replay_stepwise or wave_engine or kept_greedy"
run() {  # tool, selection, timeout
  local tool=$1 sel=$2 t=$3 extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout $t compute-sanitizer --tool $tool $extra --print-limit 50 --target-processes all \
    python -m pytest $FILES -m gpu -q -p no:cacheprovider -k "$sel" > $O/sanitize_$tool.log 2>&1
  echo "exit=$?" >> $O/sanitize_$tool.log
}
run memcheck "$ALL" 1500
run synccheck "$SMALL" 1200
run racecheck "$SMALL" 1800

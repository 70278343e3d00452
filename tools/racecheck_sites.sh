#!/bin/bash
# racecheck with every hazard printed, summarised by (kind, source line pair) -> gpurun_out/racecheck_sites.txt
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
FILES="tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_kept.py"
SEL="${1:-resample_golden_cases or staged_kernel_edge_rows or (wide_kernel_matches_oracle_and_cta_kernel and 151936-0.0) or cache_replays_reference_traces or replay_stepwise or wave_engine or kept_greedy}"
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 1000000 --target-processes all \
  python -m pytest $FILES -m gpu -q -p no:cacheprovider -k "$SEL" > $O/rc_full.log 2>&1
echo "exit=$?" > $O/racecheck_sites.txt
grep -E "SUMMARY|passed|failed" $O/rc_full.log >> $O/racecheck_sites.txt
python3 - $O/rc_full.log >> $O/racecheck_sites.txt <<'PY'
import re, sys, collections
kinds = collections.Counter()
cur = None
for line in open(sys.argv[1], errors="replace"):
    m = re.match(r"=+ (Error|Warning): (.*?) detected", line)
    if m:
        cur = [m.group(1) + ": " + m.group(2)]
        continue
    m = re.search(r"(Read|Write) Thread .* at (.*?)\+0x[0-9a-f]+ in (\S+)", line)
    if m and cur is not None:
        fn = re.sub(r"\(.*", "", m.group(2))[-60:]
        cur.append(f"{m.group(1)} {fn} {m.group(3)}")
        if len(cur) == 3:
            kinds[" | ".join(cur)] += 1
            cur = None
for k, v in kinds.most_common(40):
    print(v, k)
PY
rm -f $O/rc_full.log

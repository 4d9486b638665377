#!/usr/bin/env bash
# One GPU-box pass that produces everything profiles/ and the round's bench
# evidence need.  Run from the repo root under gpurun:
#   gpurun --timeout 2400 -- 'bash tools/profile_round.sh rNN'
# Order matters: each ncu pass runs only after the same command exited 0
# without ncu.  Outputs land in gpurun_out/<tag>/.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status"
timeout 600 ./build/compat_test > "$OUT/compat_test.log" 2>&1; echo "compat rc=$?" >> "$OUT/status"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "ref rc=$?" >> "$OUT/status"
timeout 900 python bench.py --emulate 8 > "$OUT/bench.json" 2> "$OUT/bench.err"
rc=$?; echo "bench rc=$rc" >> "$OUT/status"
python tools/timeline.py --syncs 3 --out "$OUT/timeline_1pct.txt" > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out "$OUT/timeline_10pct.txt" > /dev/null 2>&1
timeout 900 python tools/sweep.py --quick --out "$OUT/sweep.json" > "$OUT/sweep.log" 2>&1; echo "sweep rc=$?" >> "$OUT/status"
ZEN_DIAG_EXTRACT_PLAIN=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-extras > "$OUT/extract_plain.json" 2>&1
SHORT="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 600 $SHORT > "$OUT/short.json" 2> "$OUT/short.err"
rc2=$?; echo "short rc=$rc2" >> "$OUT/status"
if [ $rc2 -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file "$OUT/launches.csv" $SHORT > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?" >> "$OUT/status"
  timeout 1500 ncu --set full --clock-control none --import-source on \
      -k regex:'k_(bp_begin|extract_tiles|push_scatter|place_tiles|depth_scan|fallback|agg_mark|agg_union|agg_values|decode)' \
      -s 40 -c 10 -o "$OUT/full" $SHORT > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?" >> "$OUT/status"
fi

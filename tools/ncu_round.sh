#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for this repo, run under gpurun on ONE GPU:
#   1. the launch list of the bench command (gpu__time_duration per launch),
#   2. one `ncu --set full` capture per config kernel (tools/prof_target.py),
# each only after the same command exited 0 without ncu.
#   usage: tools/ncu_round.sh <tag> [targets...]
set -u
TAG=${1:-r01}
shift || true
TARGETS=${*:-"c5 c1 c2k4 c2k8 c3 c4"}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if [ -n "${SKIP_BENCH:-}" ]; then echo "launch list skipped";
elif timeout 900 $BENCH > $OUT/bench_plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv $BENCH > $OUT/bench_ncu.log 2>&1
  echo "launch list rc=$?"
else
  echo "bench plain run failed"; tail -20 $OUT/bench_plain.log
fi
for t in $TARGETS; do
  case $t in
    c5) K="regex:cs_hot_kernel" ;;
    c1) K="regex:cs_small" ;;
    c4) K="regex:cs_private89" ;;
    c2k4|c2k8) K="regex:hash61_key64" ;;
    c3) K="regex:pm_divmod" ;;
  esac
  if timeout 600 python tools/prof_target.py $t --reps 3 > $OUT/plain_$t.log 2>&1; then
    timeout 1200 ncu --set full --clock-control none --import-source on -k $K -s 1 -c 1 \
      -o $OUT/prof_$t python tools/prof_target.py $t --reps 3 > $OUT/ncu_$t.log 2>&1
    echo "$t ncu rc=$?"
  else
    echo "$t plain run failed"; tail -5 $OUT/plain_$t.log
  fi
done

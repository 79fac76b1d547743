set -u
mkdir -p gpurun_out
for mx in 22 23; do
  echo "== max 2^$mx items 2^31"
  MB200_SAMPLE_SHIFT=7 MB200_MAX_SAMPLE_LOG2=$mx timeout 300 python tools/prof_target.py c5 --items $((1<<31)) --reps 6 2>&1 | tail -3
done
for lg in 29 30; do
for sh in 8 7 6; do
  echo "== shift $sh items 2^$lg"
  MB200_SAMPLE_SHIFT=$sh timeout 300 python tools/prof_target.py c5 --items $((1<<lg)) --reps 6 2>&1 | tail -3
done
done

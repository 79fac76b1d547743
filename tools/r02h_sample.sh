set -u
mkdir -p gpurun_out
for sh in 8 7 6; do
 for lg in 26 28 31; do
  echo "== shift $sh items 2^$lg"
  MB200_SAMPLE_SHIFT=$sh timeout 300 python tools/prof_target.py c5 --items $((1<<lg)) --reps 5 2>&1 | tail -3
 done
done

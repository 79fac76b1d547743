set -u
mkdir -p gpurun_out
for pc in 0 8192 4096 2048; do
  echo "== per_cta $pc"
  MB200_COUNT_PER_CTA=$pc timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnt_$pc.csv python tools/prof_target.py c5 --items $((1<<31)) --reps 2 > gpurun_out/cnt_$pc.log 2>&1; echo "ncu rc=$?"
  python tools/launches.py gpurun_out/cnt_$pc.csv | tail -7 | head -5
  grep "hot set" gpurun_out/cnt_$pc.log
done

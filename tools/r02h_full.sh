set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fixed_launches_31.csv python tools/prof_target.py c5 --items $((1<<31)) --reps 2 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/fixed_launches_31.csv | tail -9

# fixed per-call cost of the config-5 pipeline: shard sizes 2^22..2^31, event times and the serialised launch list
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "hot or heavy or zipf or c5 or sketch" > gpurun_out/hot_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/hot_tests.log
for lg in 22 28 31; do
  timeout 300 python tools/prof_target.py c5 --items $((1<<lg)) --reps 6 > gpurun_out/fixed_$lg.log 2>&1; echo "2^$lg rc=$?"; tail -3 gpurun_out/fixed_$lg.log
done
for lg in 28 31; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/fixed_launches_$lg.csv python tools/prof_target.py c5 --items $((1<<lg)) --reps 2 > /dev/null 2>&1; echo "ncu 2^$lg rc=$?"
done
python tools/launches.py gpurun_out/fixed_launches_31.csv | tail -10
python tools/launches.py gpurun_out/fixed_launches_28.csv | tail -10

# quick GPU check used while iterating: parity tests of the touched paths, event
# timings of the config kernels, and the launch list of config 5 / config 4
K=${K:-"hot or sketch or cpp or hash or c1 or golden"}
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/t1.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t1.log
for t in ${TARGETS:-c5 c4}; do python tools/prof_target.py $t --reps 3; done
if [ -z "${NO_NCU:-}" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5.csv python tools/prof_target.py c5 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l4.csv python tools/prof_target.py c4 --reps 1 > /dev/null 2>&1
fi
echo done

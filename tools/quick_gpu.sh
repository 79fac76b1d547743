timeout 600 python -m pytest tests -m gpu -x -q -k "hot or sketch or cpp" > gpurun_out/t1.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/t1.log
python tools/prof_target.py c5 --reps 3; python tools/prof_target.py c4 --reps 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5.csv python tools/prof_target.py c5 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l4.csv python tools/prof_target.py c4 --reps 1 > /dev/null 2>&1
echo done

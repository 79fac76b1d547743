# fresh-box check: GPU tests, smoke, bench, shard launch list
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python tools/prof_target.py c5 --items $((1<<28)) --reps 5 > gpurun_out/shard.log 2>&1; echo "shard rc=$?"; cat gpurun_out/shard.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shard_launches.csv python tools/prof_target.py c5 --items $((1<<28)) --reps 2 > /dev/null 2>&1; echo "ncu rc=$?"

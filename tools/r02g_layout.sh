# shard (2^28) vs full-stream prepass: hot-set stats, ncu of layout and count kernels
set -u
mkdir -p gpurun_out/r02g
for n in $((1<<28)) $((1<<31)); do
  timeout 300 python tools/prof_target.py c5 --items $n --reps 3 > gpurun_out/r02g/plain_$n.log 2>&1; echo "plain $n rc=$?"; cat gpurun_out/r02g/plain_$n.log
done
for k in hh_layout hh_count hh_select; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r02g/prof_$k python tools/prof_target.py c5 --items $((1<<28)) --reps 2 > gpurun_out/r02g/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done

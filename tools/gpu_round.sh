set -u
python tools/imad_probe.py > gpurun_out/imad_probe_r02f.txt 2>&1
bash tools/ncu_round.sh r02f > gpurun_out/ncu_round_r02f.log 2>&1
python tools/make_profiles.py r02f > gpurun_out/mkprof_r02f.log 2>&1
mkdir -p gpurun_out/profiles_r02f && cp -r profiles/r02f/. gpurun_out/profiles_r02f/ && cp profiles/ncu_traffic.json gpurun_out/profiles_r02f/ncu_traffic_root.json
rm -f gpurun_out/ncu_r02f/*.ncu-rep
python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
echo done

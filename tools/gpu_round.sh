# One measurement round on the GPU box: IMAD peak probe, launch list + ncu --set full per config
# (tools/ncu_round.sh), summaries into profiles/<tag> (tools/make_profiles.py), then the bench line.
#   usage: bash tools/gpu_round.sh <tag>
set -u
TAG=${1:-r02h}
python tools/imad_probe.py > gpurun_out/imad_probe_$TAG.txt 2>&1
bash tools/ncu_round.sh $TAG > gpurun_out/ncu_round_$TAG.log 2>&1
python tools/make_profiles.py $TAG > gpurun_out/mkprof_$TAG.log 2>&1
mkdir -p gpurun_out/profiles_$TAG && cp -r profiles/$TAG/. gpurun_out/profiles_$TAG/ && cp profiles/ncu_traffic.json gpurun_out/profiles_$TAG/ncu_traffic_root.json
rm -f gpurun_out/ncu_$TAG/*.ncu-rep
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo done

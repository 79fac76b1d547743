#!/bin/bash
# e2e stall diagnosis on the GPU box: host memory / CPU state around the
# host-buffer CountSketch::process steps (bench.py e2e leg and tools/e2e_probe.py)
mkdir -p gpurun_out/e2e_diag
D=gpurun_out/e2e_diag
(free -g; nproc; cat /proc/meminfo | head -20; cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/defrag) > $D/host.txt 2>&1
vmstat -t 1 > $D/vmstat.txt 2>&1 &
VM=$!
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $D/bench.log 2>&1
echo "bench rc=$?"
timeout 300 python tools/e2e_probe.py > $D/probe.log 2>&1
echo "probe rc=$?"
kill $VM
python - <<'PY'
import json
L=open('gpurun_out/e2e_diag/bench.log').read().strip().split('\n')[-1]
d=json.loads(L)
print('e2e', d['e2e']['value'], [round(x) for x in d['e2e']['step_ms']])
PY
tail -5 $D/probe.log

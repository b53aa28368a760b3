#!/bin/bash
# quick loop: GPU parity, per-kernel timings, one ncu capture of the tile kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_kernels.py --steps 60 >> gpurun_out/kern.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_srdct_tiles}" -s 2 -c 2 -o gpurun_out/prof_$TAG python tools/profile_c2.py --steps 8 > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu1.log
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/kern.log; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'phases',d['solve']['phases_ms'])
    print({k:round(v['avg_us'],2) for k,v in d['kernels'].items()})
PY
tail -n 2 gpurun_out/ncu1.log

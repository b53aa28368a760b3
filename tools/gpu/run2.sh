#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sell_spmv|k_update|k_srdct256" -s 3 -c 3 -o gpurun_out/prof_c2 python tools/profile_c2.py --steps 8 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
tail -25 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench.log; tail -5 gpurun_out/ncu.log

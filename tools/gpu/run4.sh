#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SDR_FUSE=0 timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_nofuse.log 2>&1; echo "pytest nofuse rc=$?" >> gpurun_out/pytest_gpu_nofuse.log
for f in 0 1; do SDR_FUSE=$f timeout 300 python tools/bench_kernels.py --steps 60 >> gpurun_out/kern.log 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sell_spmv|k_update" -s 3 -c 2 -o gpurun_out/prof_c2c python tools/profile_c2.py --steps 8 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu_nofuse.log; cat gpurun_out/kern.log; tail -c 3000 gpurun_out/bench.log; tail -2 gpurun_out/ncu.log

#!/bin/bash
# uniform-D SELL-DIA with prefetched offsets: parity (DIA on/off), kernel timings, K1 ncu.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SDR_DIA=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu_nodia.log 2>&1; echo "pytest nodia rc=$?" >> gpurun_out/pytest_gpu_nodia.log
for d in 0 1; do echo "SDR_DIA=$d" >> gpurun_out/kern.log; SDR_DIA=$d timeout 300 python tools/bench_kernels.py --steps 60 >> gpurun_out/kern.log 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_srdct_tiles|k_sell_spmv" -s 4 -c 3 -o gpurun_out/prof_us_v3 python tools/profile_c2.py --steps 8 > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu1.log
tail -3 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu_nodia.log; cat gpurun_out/kern.log; tail -c 2500 gpurun_out/bench.log; tail -n 2 gpurun_out/ncu1.log

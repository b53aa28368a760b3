#!/bin/bash
# K1 SELL vs SELL-DIA: plain timings, then one ncu --set full capture of each.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for d in 0 1; do echo "SDR_DIA=$d" >> gpurun_out/kern.log; SDR_DIA=$d timeout 300 python tools/bench_kernels.py --steps 60 >> gpurun_out/kern.log 2>&1; done
for d in 0 1; do
SDR_DIA=$d timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain$d.log 2>&1 && \
SDR_DIA=$d timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sell_spmv" -s 4 -c 1 -o gpurun_out/prof_k1_dia$d python tools/profile_c2.py --steps 8 > gpurun_out/ncu$d.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu$d.log
done
cat gpurun_out/kern.log; tail -2 gpurun_out/ncu*.log

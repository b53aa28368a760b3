#!/bin/bash
# Round profile capture: full ncu of K1 / K2 and of the recycle product, the
# bench launch list, a default bench line. Each ncu run follows a clean run of
# the same command.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 300 python tools/profile_c2.py --steps 8 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sell_spmv|k_srdct_tiles" -s 4 -c 2 -o gpurun_out/${TAG}_full python tools/profile_c2.py --steps 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 300 python tools/profile_c2.py --steps 2 --solve > gpurun_out/prof_solve.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgemm" -c 1 -o gpurun_out/${TAG}_rgemm python tools/profile_c2.py --steps 2 --solve > gpurun_out/ncu_rgemm.log 2>&1; echo "ncu rgemm rc=$?" >> gpurun_out/ncu_rgemm.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
tail -c 3000 gpurun_out/bench_default.log; tail -n 2 gpurun_out/ncu_full.log gpurun_out/ncu_rgemm.log gpurun_out/ncu_launch.log

#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
SDR_TRACE=1 timeout 300 python tools/trace_tiles.py > gpurun_out/trace.log 2>&1; echo "rc=$?" >> gpurun_out/trace.log
cat gpurun_out/trace.log

#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
WG_FENCE_SCOPE=sys timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rA -k "mg" > gpurun_out/r2y_mg_sys.log 2>&1; echo "sys rc=$?"; tail -2 gpurun_out/r2y_mg_sys.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rA -k "mg" > gpurun_out/r2y_mg_default.log 2>&1; echo "default rc=$?"; tail -2 gpurun_out/r2y_mg_default.log

#!/bin/bash
# compute-sanitizer, one tool per gpurun call (B200_PROFILING.md): tools/gpu_sanitize.sh racecheck|synccheck|memcheck
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=$1
timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_case.py > gpurun_out/sanitize_$T.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/sanitize_$T.log

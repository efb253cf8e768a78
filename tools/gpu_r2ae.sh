#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA -k "not mg" > gpurun_out/r2ae_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2ae_tests.log
{
bash tools/ab_env.sh 2 "-" --S 8
bash tools/ab_env.sh 4 "-" --S 8
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2
} > gpurun_out/r2ae_ab.txt 2>&1; cat gpurun_out/r2ae_ab.txt

#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
{
bash tools/ab_env.sh 4 "-|WG_HIER=1 WG_MG=0|WG_HIER=1 WG_MG=1" --S 8
bash tools/ab_env.sh 4 "-|WG_HIER=1 WG_MG=0" --S 4
bash tools/ab_env.sh 2 "-|WG_HIER=1 WG_MG=0" --S 8
} > gpurun_out/r2af_ab.txt 2>&1; cat gpurun_out/r2af_ab.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA -x -k "nvl-hier" > gpurun_out/r2af_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2af_tests.log

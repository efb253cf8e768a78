#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
{
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_cpa.so ab/lib_t5.so ab/lib_t2.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_cpa.so ab/lib_t5.so ab/lib_t2.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_cpa.so" --S 4
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_cpa.so" --P 2 --S 2
} > gpurun_out/r2ah.txt 2>&1; cat gpurun_out/r2ah.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA -x -k "not mg" > gpurun_out/r2ah_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/r2ah_tests.log

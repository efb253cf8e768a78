#!/bin/bash
# hierarchical sums in the pull kernel (WG_HIER=1 WG_MG=0) with deeper producer rings, 2 and 4 GPUs
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
export WG_HIER=1 WG_MG=0
{
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_nd5.so ab/lib_nd6.so ab/lib_nd8.so ab/lib_nd10.so" --S 8
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_nd6.so ab/lib_nd8.so" --S 4
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_nd5.so ab/lib_nd6.so ab/lib_nd8.so ab/lib_nd10.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_nd6.so ab/lib_nd8.so" --S 4
} > gpurun_out/r2ab.txt 2>&1
cat gpurun_out/r2ab.txt

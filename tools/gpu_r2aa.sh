#!/bin/bash
# split-kernel producer depth / local-leaf TMA A/B at 2 and 4 GPUs (P=8 S=8) and 4 GPUs S=4
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
{
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_d5.so ab/lib_tl0.so ab/lib_d6tl0.so ab/lib_d8tl0.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_d5.so ab/lib_tl0.so ab/lib_d6tl0.so ab/lib_d8tl0.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_d5.so ab/lib_d6tl0.so" --S 4
} > gpurun_out/r2aa.txt 2>&1
cat gpurun_out/r2aa.txt

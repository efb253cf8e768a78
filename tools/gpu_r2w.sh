#!/bin/bash
# 1-GPU A/B of local-kernel build variants (two passes to see the run-to-run spread)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for pass in 1 2; do
  bash tools/ab_single.sh "ab/lib_default.so ab/lib_t4s.so ab/lib_w8.so ab/lib_nocs.so ab/lib_noef.so ab/lib_t1w8.so"
done > gpurun_out/r2w_ab.txt 2>&1
cat gpurun_out/r2w_ab.txt

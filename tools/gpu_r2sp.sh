#!/bin/bash
# Phase profile of the split kernel (WG_PROF_COUNTERS build) at 2 and 4 GPUs, P=8 S=8
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for N in 2 4; do
WAGMA_B200_LIB=$PWD/ab/lib_prof.so WG_PROF_SPLIT=1 WG_PROF_DUMP=gpurun_out/sp$N timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N tools/phase_profile.py --S 8 --iters 2 > gpurun_out/sp_prof_$N.txt 2>&1
tail -3 gpurun_out/sp_prof_$N.txt
done

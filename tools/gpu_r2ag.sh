#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
WAGMA_B200_LIB=$PWD/ab/lib_prof.so WG_PROF_SPLIT=1 WG_PROF_DUMP=gpurun_out/sph4 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/sph_prof_4.txt 2>&1
WAGMA_B200_LIB=$PWD/ab/lib_prof.so WG_PROF_DUMP=gpurun_out/nvh2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/nvh_prof_2.txt 2>&1
tail -2 gpurun_out/sph_prof_4.txt gpurun_out/nvh_prof_2.txt

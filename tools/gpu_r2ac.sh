#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
export WG_HIER=1 WG_MG=1
{
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_nself.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so ab/lib_nself.so" --S 8
bash tools/ab_multi2.sh 4 "ab/lib_default.so" --S 4
} > gpurun_out/r2ac.txt 2>&1
cat gpurun_out/r2ac.txt
WG_PROF_MG=1 WG_PROF_DUMP=gpurun_out/r2ac_prof4 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2ac_prof_mg4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "mg and (baseline or stress)" > gpurun_out/r2ac_tests.log 2>&1; tail -2 gpurun_out/r2ac_tests.log

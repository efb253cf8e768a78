cd $GRAFT_REPO_ROOT
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_acq0.so ab/lib_pb4.so" --S 8 > gpurun_out/r2l_ab.txt 2>&1
WG_PROF_MG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2l_prof.txt 2>&1
cat gpurun_out/r2l_ab.txt; tail -2 gpurun_out/r2l_prof.txt

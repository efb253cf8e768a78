cd $GRAFT_REPO_ROOT
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_dl0.so ab/lib_dli2.so" --S 8 > gpurun_out/r2n_ab.txt 2>&1
bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 4 >> gpurun_out/r2n_ab.txt 2>&1
WG_MG=0 bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 8 >> gpurun_out/r2n_ab.txt 2>&1
mkdir -p gpurun_out/prof; WG_PROF_DUMP=gpurun_out/prof/mgd WG_PROF_MG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2n_prof.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "mg" > gpurun_out/r2n_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_multi.log
cat gpurun_out/r2n_ab.txt; tail -3 gpurun_out/r2n_multi.log

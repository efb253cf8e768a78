cd $GRAFT_REPO_ROOT
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_i4.so ab/lib_i2.so" --S 8 > gpurun_out/r2k_ab.txt 2>&1
bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 4 >> gpurun_out/r2k_ab.txt 2>&1
WG_PROF_MG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2k_prof.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2k_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_multi.log
cat gpurun_out/r2k_ab.txt; tail -2 gpurun_out/r2k_prof.txt; tail -3 gpurun_out/r2k_multi.log

cd $GRAFT_REPO_ROOT
bash tools/ab_single.sh "ab/lib_stack.so ab/lib_st0.so ab/lib_st_t4.so ab/lib_st_t1.so ab/lib_stack.so ab/lib_st0.so" > gpurun_out/r2g_ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_multi.py > gpurun_out/r2g_gpu1.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_gpu1.log
cat gpurun_out/r2g_ab.txt; tail -3 gpurun_out/r2g_gpu1.log

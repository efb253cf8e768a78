cd $GRAFT_REPO_ROOT
for S in 8 4; do bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_mgl4.so ab/lib_mgl6.so ab/lib_mgi4.so" --S $S; done > gpurun_out/r2f_ab.txt 2>&1
WG_MG=0 bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 8 >> gpurun_out/r2f_ab.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_metrics.py -q -x > gpurun_out/r2f_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_multi.log
cat gpurun_out/r2f_ab.txt; tail -3 gpurun_out/r2f_multi.log

cd $GRAFT_REPO_ROOT
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_dli2.so" --S 8 > gpurun_out/r2o_ab.txt 2>&1
bash tools/ab_multi2.sh 2 "ab/lib_default.so ab/lib_dli2.so" --S 4 >> gpurun_out/r2o_ab.txt 2>&1
WG_MG=0 bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 8 >> gpurun_out/r2o_ab.txt 2>&1
WG_HIER=0 bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 8 >> gpurun_out/r2o_ab.txt 2>&1
WG_ADAPTIVE_GRACE=0 bash tools/ab_multi2.sh 2 "ab/lib_default.so" --S 8 >> gpurun_out/r2o_ab.txt 2>&1
cat gpurun_out/r2o_ab.txt

cd $GRAFT_REPO_ROOT
CMD="python bench.py --no-cpu --no-e2e --steps 3 --warmup 3"
$CMD > gpurun_out/r2d_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wagma_local -s 3 -c 1 -o gpurun_out/r2d_local $CMD > gpurun_out/r2d_ncu.log 2>&1
WAGMA_B200_LIB=$PWD/ab/lib_w16.so $CMD > gpurun_out/r2d_plain16.log 2>&1 && WAGMA_B200_LIB=$PWD/ab/lib_w16.so ncu --set full --clock-control none --import-source on -k regex:wagma_local -s 3 -c 1 -o gpurun_out/r2d_local16 $CMD > gpurun_out/r2d_ncu16.log 2>&1
tail -2 gpurun_out/r2d_ncu.log gpurun_out/r2d_ncu16.log

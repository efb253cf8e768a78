cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2b_gpu.log
bash tools/ab_single.sh "ab/lib_default.so ab/lib_t1.so ab/lib_w16.so ab/lib_t1w4.so ab/lib_ef.so ab/lib_cs.so ab/lib_efcs.so ab/lib_default.so" > gpurun_out/r2b_ab.txt 2>&1
CMD="python bench.py --no-cpu --no-e2e --steps 3 --warmup 3"
$CMD > gpurun_out/r2b_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wagma_local -s 3 -c 1 -o gpurun_out/r2b_local $CMD > gpurun_out/r2b_ncu.log 2>&1
tail -3 gpurun_out/r2b_gpu.log; cat gpurun_out/r2b_ab.txt; tail -3 gpurun_out/r2b_ncu.log

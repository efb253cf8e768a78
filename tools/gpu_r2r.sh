cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_faults.py tests/test_gpu_api.py -q -x > gpurun_out/r2r_tests.log 2>&1; tail -3 gpurun_out/r2r_tests.log
timeout 300 python -m pytest tests/test_gpu_multi.py -q -x -k "mismatched" > gpurun_out/r2r_multi.log 2>&1; tail -3 gpurun_out/r2r_multi.log
{
bash tools/ab_env.sh 2 "-|WG_MG_NSI_MAX=3|WG_FENCE_SCOPE=sys" --S 8
bash tools/ab_env.sh 4 "-|WG_FENCE_SCOPE=sys" --S 8
} > gpurun_out/r2r_ab.txt 2>&1
WG_PROF_MG=1 WG_PROF_DUMP=gpurun_out/r2r_prof2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2r_prof_mg2.txt 2>&1
WG_PROF_MG=1 WG_PROF_DUMP=gpurun_out/r2r_prof4 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2r_prof_mg4.txt 2>&1
cat gpurun_out/r2r_ab.txt; tail -2 gpurun_out/r2r_prof_mg2.txt; tail -2 gpurun_out/r2r_prof_mg4.txt

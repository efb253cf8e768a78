cd $GRAFT_REPO_ROOT
{
bash tools/ab_env.sh 2 "-|WG_MG_NSI_MAX=3" --S 8
bash tools/ab_env.sh 2 "-" --S 4
bash tools/ab_env.sh 4 "-|WG_MG_NSI_MAX=4|WG_MG_NSI_MAX=3" --S 8
bash tools/ab_env.sh 4 "-" --S 4
} > gpurun_out/r2q_ab.txt 2>&1
cp gpurun_out/ab_e.log gpurun_out/r2q_last.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "mg" > gpurun_out/r2q_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_multi.log
WG_PROF_MG=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2q_prof_mg4.txt 2>&1
cat gpurun_out/r2q_ab.txt; tail -3 gpurun_out/r2q_multi.log; tail -3 gpurun_out/r2q_prof_mg4.txt

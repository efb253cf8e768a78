cd $GRAFT_REPO_ROOT
nvidia-smi nvlink -h > gpurun_out/r2p_nvlink_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r2p_nvlink_gt.txt 2>&1
nvidia-smi topo -m > gpurun_out/r2p_topo.txt 2>&1
{
bash tools/ab_env.sh 2 "-|WG_MG=0|WG_HIER=0|WG_ADAPTIVE_GRACE=0" --S 8
bash tools/ab_env.sh 2 "-|WG_HIER=0" --S 4
bash tools/ab_env.sh 4 "WG_MG=0|WG_HIER=0" --S 8
bash tools/ab_env.sh 4 "-|WG_MG=0|WG_HIER=0" --S 4
} > gpurun_out/r2p_ab.txt 2>&1
mkdir -p gpurun_out/prof
WG_PROF_MG=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2p_prof_mg.txt 2>&1
cat gpurun_out/r2p_ab.txt; tail -4 gpurun_out/r2p_prof_mg.txt

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
WG_PROF_DUMP=gpurun_out/prof/mg WG_PROF_MG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2m_prof.txt 2>&1
WG_MG=0 WG_PROF_DUMP=gpurun_out/prof/nvl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2m_prof_nvl.txt 2>&1
ls gpurun_out/prof; tail -2 gpurun_out/r2m_prof_nvl.txt

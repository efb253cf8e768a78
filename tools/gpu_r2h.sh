cd $GRAFT_REPO_ROOT
WG_PROF_MG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 4 > gpurun_out/r2h_prof.txt 2>&1
bash tools/gpu_r2g.sh
tail -8 gpurun_out/r2h_prof.txt

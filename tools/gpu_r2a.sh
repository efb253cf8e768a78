cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2a_kern.log 2>&1; echo "kern rc=$?" >> gpurun_out/r2a_kern.log
WG_LOC=0 timeout 300 python bench.py --no-cpu --no-e2e --steps 200 > gpurun_out/r2a_b_old.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 200 > gpurun_out/r2a_b_new.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/r2a_gpu.log
tail -3 gpurun_out/r2a_kern.log gpurun_out/r2a_gpu.log; tail -c 600 gpurun_out/r2a_b_old.log; tail -c 600 gpurun_out/r2a_b_new.log

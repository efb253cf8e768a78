#!/bin/bash
# Multi-GPU parity suite twice on 4 GPUs: default (GPU-scope flag fences) and the strictly PTX-scoped WG_FENCE_SCOPE=sys.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2x_gpus.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA > gpurun_out/r2x_multi_default.log 2>&1; echo "default rc=$?"; tail -2 gpurun_out/r2x_multi_default.log
WG_FENCE_SCOPE=sys timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rA > gpurun_out/r2x_multi_sys.log 2>&1; echo "sys rc=$?"; tail -2 gpurun_out/r2x_multi_sys.log

for L in ${PP_LIBS:-base sd5}; do
WAGMA_B200_LIB=$PWD/ab/lib_$L.so WG_PROF_DUMP=gpurun_out/prof/$L WG_PROF_SPLIT=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 tools/phase_profile.py --iters 2 ${PP_ARGS} > gpurun_out/phase_$L.log 2>&1
done

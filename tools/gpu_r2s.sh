cd $GRAFT_REPO_ROOT
for L in ab/lib_g1.so ab/lib_nosync.so ab/lib_default.so; do
  WAGMA_B200_LIB=$PWD/$L timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29613 bench.py --gpus 4 --steps 30 --warmup 5 --no-e2e > gpurun_out/r2s_$(basename $L).log 2>&1
  echo "$L rc=$? $(tail -1 gpurun_out/r2s_$(basename $L).log | cut -c1-150)"
  grep -m2 -i 'illegal\|error' gpurun_out/r2s_$(basename $L).log
done
python tools/nvml_nvlink.py 0 1 > gpurun_out/r2s_nvml.txt 2>&1; cat gpurun_out/r2s_nvml.txt

cd $GRAFT_REPO_ROOT
for L in ab/lib_default.so ab/lib_gp4.so ab/lib_gr4.so ab/lib_nodirect.so; do
  WAGMA_B200_LIB=$PWD/$L timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29613 bench.py --gpus 4 --steps 100 --warmup 5 --no-e2e > gpurun_out/r2t_4_$(basename $L).log 2>&1
  echo "N=4 S=8 $L rc=$? $(tail -1 gpurun_out/r2t_4_$(basename $L).log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3))' 2>&1 | tail -1)"
  grep -m1 -i 'illegal' gpurun_out/r2t_4_$(basename $L).log
done
for L in ab/lib_default.so ab/lib_gp4.so ab/lib_nodirect.so; do
  WAGMA_B200_LIB=$PWD/$L timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29614 bench.py --gpus 2 --steps 100 --warmup 5 --no-e2e > gpurun_out/r2t_2_$(basename $L).log 2>&1
  echo "N=2 S=8 $L rc=$? $(tail -1 gpurun_out/r2t_2_$(basename $L).log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3))' 2>&1 | tail -1)"
done
WG_PROF_MG=1 WG_PROF_DUMP=gpurun_out/r2t_prof2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2t_prof_mg2.txt 2>&1
WG_PROF_MG=1 WG_PROF_DUMP=gpurun_out/r2t_prof4 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 tools/phase_profile.py --S 8 --iters 2 > gpurun_out/r2t_prof_mg4.txt 2>&1

#!/bin/bash
# Round-2 N=1 evidence: bench line, then the same command's ncu launch list and one --set full capture of the local kernel.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2u_bench_n1.json 2> gpurun_out/r2u_bench_n1.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2u_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2u_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2u_ncu_list.log 2>&1; echo "list rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2u_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wagma_local -s 3 -c 1 -f \
  -o gpurun_out/r2u_local_full python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2u_ncu_full.log 2>&1; echo "full rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2u_bench_n1.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"

#!/bin/bash
# Round-end evidence on one GPU: bench line, reference arm, ncu launch list, one ncu --set full capture.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/reference.json 2> gpurun_out/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wagma_step -s 3 -c 1 -f \
  -o gpurun_out/step_full python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo done

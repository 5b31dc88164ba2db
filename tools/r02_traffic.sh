#!/bin/bash
# DRAM bytes of every inner-kernel launch of one cfg5 64-RHS step (ncu metrics pass) -> gpurun_out/traffic.csv;
# tools/ncu_traffic.py turns it into profiles/r02_traffic.json (bench.py's roofline.traffic)
mkdir -p gpurun_out
timeout 2400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base \
    --profile-from-start off -k regex:inner_items_kernel --csv --log-file gpurun_out/traffic.csv \
    python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic.log 2>&1
echo "traffic exit $?" >> gpurun_out/traffic.log

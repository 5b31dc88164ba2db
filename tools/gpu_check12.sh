#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/c12_bench_cellmajor.json 2> gpurun_out/c12_bench_cellmajor.err
PT_K1_COLMAJOR=1 timeout 600 $B > gpurun_out/c12_bench_colmajor.json 2> gpurun_out/c12_bench_colmajor.err
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 --no-extras --no-cpu-baseline --e2e-steps 2 > gpurun_out/c12_cfg2.json 2> gpurun_out/c12_cfg2.err
timeout 600 python tools/offline_times.py cfg5 k1 > gpurun_out/c12_offline.log 2>&1

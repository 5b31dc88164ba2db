#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/c10_bench_epi.json 2> gpurun_out/c10_bench_epi.err
timeout 600 $B --nrhs 1 > gpurun_out/c10_bench1_epi.json 2> gpurun_out/c10_bench1_epi.err
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "item or default" > gpurun_out/c10_paths.log 2>&1; echo "exit $?" >> gpurun_out/c10_paths.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "(fixture and (cfg4 or cfg5)) or histogram" > gpurun_out/c10_parity.log 2>&1; echo "exit $?" >> gpurun_out/c10_parity.log

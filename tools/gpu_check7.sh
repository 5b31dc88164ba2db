#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/c7_bench_kc64.json 2> gpurun_out/c7_bench_kc64.err
PT_SG_KC=32 timeout 600 $B > gpurun_out/c7_bench_kc32.json 2> gpurun_out/c7_bench_kc32.err
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "stage-gemm" > gpurun_out/c7_paths.log 2>&1; echo "exit $?" >> gpurun_out/c7_paths.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "batched and (cfg3 or cfg4)" > gpurun_out/c7_batched.log 2>&1; echo "exit $?" >> gpurun_out/c7_batched.log

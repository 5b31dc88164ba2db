#!/bin/bash
# quick GPU regression for the streaming stage GEMM and the K1-built offline operators, then A/B timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "offline_operators" > gpurun_out/c2_offline.log 2>&1; echo "exit $?" >> gpurun_out/c2_offline.log
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "stage-gemm or default" > gpurun_out/c2_paths.log 2>&1; echo "exit $?" >> gpurun_out/c2_paths.log
timeout 600 python -m pytest tests/test_dist_gloo.py -x -q > gpurun_out/c2_dist.log 2>&1; echo "exit $?" >> gpurun_out/c2_dist.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --durations=8 -k "batched and (cfg2 or cfg3 or cfg5)" > gpurun_out/c2_batched.log 2>&1; echo "exit $?" >> gpurun_out/c2_batched.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/c2_bench_sgemm.json 2> gpurun_out/c2_bench_sgemm.err
PT_NO_SGEMM=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/c2_bench_nosgemm.json 2> gpurun_out/c2_bench_nosgemm.err
tail -3 gpurun_out/c2_*.log

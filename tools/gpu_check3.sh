#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --durations=8 -k "batched and (cfg4 or cfg5)" > gpurun_out/c3_batched.log 2>&1; echo "exit $?" >> gpurun_out/c3_batched.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_bench_sgemm.json 2> gpurun_out/c3_bench_sgemm.err
PT_NO_SGEMM=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_bench_nosgemm.json 2> gpurun_out/c3_bench_nosgemm.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync_micro tools/gridsync_micro.cu && /tmp/gridsync_micro > gpurun_out/c3_gridsync.log 2>&1
tail -3 gpurun_out/c3_*.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/b256_cfg4.json 2> gpurun_out/b256_cfg4.err
PT_BATCH_RHS=64 timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/b64_cfg4.json 2> gpurun_out/b64_cfg4.err
PT_BATCH_RHS=128 timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/b128_cfg4.json 2> gpurun_out/b128_cfg4.err
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "batched and cfg4" > gpurun_out/b256_tests.log 2>&1; echo "exit $?" >> gpurun_out/b256_tests.log

#!/bin/bash
# last check of the round: the new multi-batch test, smoke(), the bench line and the reference arm
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "lockstep_batch or plr" > gpurun_out/final_tests.log 2>&1; echo "exit $?" >> gpurun_out/final_tests.log
timeout 600 python __graft_entry__.py > gpurun_out/final_smoke.log 2>&1; echo "exit $?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "exit $?" >> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err

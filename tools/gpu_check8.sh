#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "item or default" > gpurun_out/c8_paths.log 2>&1; echo "exit $?" >> gpurun_out/c8_paths.log
timeout 600 $B > gpurun_out/c8_bench_bdir.json 2> gpurun_out/c8_bench_bdir.err
PT_II_DBG=64 timeout 600 $B > gpurun_out/c8_bench_nobdir.json 2> gpurun_out/c8_bench_nobdir.err
timeout 600 $B --nrhs 1 > gpurun_out/c8_bench1_bdir.json 2> gpurun_out/c8_bench1_bdir.err
PT_NO_SCAN=1 timeout 600 $B > gpurun_out/c8_bench_bdir_noscan.json 2> gpurun_out/c8_bench_bdir_noscan.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "(fixture and (cfg4 or cfg5)) or (batched and (cfg4 or cfg5)) or histogram" > gpurun_out/c8_parity.log 2>&1; echo "exit $?" >> gpurun_out/c8_parity.log

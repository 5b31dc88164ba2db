#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
PT_V1_SCAN_R=8 timeout 600 $B --nrhs 1 > gpurun_out/c9_bench1_v1scan.json 2> gpurun_out/c9_bench1_v1scan.err
PT_V1_SCAN_R=8 timeout 600 $B --nrhs 8 > gpurun_out/c9_bench8_v1scan.json 2> gpurun_out/c9_bench8_v1scan.err
PT_V1_SCAN_R=8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fixture and (cfg4 or cfg5)" > gpurun_out/c9_parity.log 2>&1; echo "exit $?" >> gpurun_out/c9_parity.log
bash tools/r02_traffic.sh

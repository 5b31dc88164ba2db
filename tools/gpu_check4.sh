#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "item or default" > gpurun_out/c4_paths.log 2>&1; echo "exit $?" >> gpurun_out/c4_paths.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --durations=8 -k "(fixture and (cfg4 or cfg5)) or (batched and (cfg4 or cfg5))" > gpurun_out/c4_parity.log 2>&1; echo "exit $?" >> gpurun_out/c4_parity.log
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/c4_bench_scan.json 2> gpurun_out/c4_bench_scan.err
PT_NO_SCAN=1 timeout 600 $B > gpurun_out/c4_bench_noscan.json 2> gpurun_out/c4_bench_noscan.err
timeout 600 $B --nrhs 1 > gpurun_out/c4_bench1_default.json 2> gpurun_out/c4_bench1_default.err
PT_ITEMS_ALL=1 timeout 600 $B --nrhs 1 > gpurun_out/c4_bench1_all_scan.json 2> gpurun_out/c4_bench1_all_scan.err
PT_ITEMS_ALL=1 PT_NO_SCAN=1 timeout 600 $B --nrhs 1 > gpurun_out/c4_bench1_all_noscan.json 2> gpurun_out/c4_bench1_all_noscan.err
PT_ITEMS_ALL=1 timeout 600 $B --nrhs 8 > gpurun_out/c4_bench8_all_scan.json 2> gpurun_out/c4_bench8_all_scan.err
timeout 600 $B --nrhs 8 > gpurun_out/c4_bench8_default.json 2> gpurun_out/c4_bench8_default.err
tail -3 gpurun_out/c4_*.log

#!/bin/bash
# quick GPU regression: parity against the fixtures (small cases, cfg1-3), graph replay, then the bench line
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fixture and not cfg4 and not cfg5 or repeated" > gpurun_out/chk_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/chk_tests.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/chk_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/chk_bench.log

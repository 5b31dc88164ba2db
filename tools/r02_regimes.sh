#!/bin/bash
# The other north-star regimes (one bench line each, appended to gpurun_out/regimes.jsonl):
#   gpurun --timeout 3000 -- bash tools/r02_regimes.sh
mkdir -p gpurun_out
: > gpurun_out/regimes.jsonl
run() { timeout 900 python bench.py --no-extras --no-cpu-baseline --e2e-steps 2 "$@" >> gpurun_out/regimes.jsonl 2>> gpurun_out/regimes.err; }
run --config cfg2 --nrhs 1 --steps 20 --warmup 5
run --config cfg2 --steps 20 --warmup 5
run --config cfg3 --nrhs 1 --steps 5 --warmup 3
run --config cfg3 --steps 5 --warmup 3
run --config cfg4 --steps 2 --warmup 1
run --config cfg4 --nrhs 64 --steps 2 --warmup 1
run --config cfg5 --nrhs 1 --steps 3 --warmup 1
run --config cfg5 --nrhs 8 --steps 3 --warmup 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "plr or reference_objects" > gpurun_out/regimes_tests.log 2>&1; echo "exit $?" >> gpurun_out/regimes_tests.log
wc -l gpurun_out/regimes.jsonl

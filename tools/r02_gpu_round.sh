#!/bin/bash
# Round-2 GPU evidence in one gpurun call: GPU tests, the bench line, the reference arm, the ncu launch list of
# the bench's timed region and one `--set full` capture of the dominant kernels (with the DMMA sub-pipe metric).
#   gpurun --timeout 3000 -- bash tools/r02_gpu_round.sh [tests] [bench] [ref] [launches] [full]
mkdir -p gpurun_out
what="${*:-tests bench ref launches full}"
DM="sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for w in $what; do
case $w in
tests)
  timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/tests.log 2>&1
  echo "tests exit $?" >> gpurun_out/tests.log ;;
bench)
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err ;;
ref)
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "ref exit $?" >> gpurun_out/bench_ref.err ;;
launches)
  # the bench command's timed region (cudaProfilerStart/Stop bracket it), one step
  timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off \
      --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches.log 2>&1
  echo "launches exit $?" >> gpurun_out/launches.log ;;
full)
  # cfg5 64 RHS: a few launches of each hot kernel from the middle of the timed solve
  for k in inner_items_kernel k_stage_gemm k1_twisted; do
    skip=40; [ $k = k1_twisted ] && skip=0
    timeout 1200 ncu --set full --metrics $DM --clock-control none --import-source on --profile-from-start off \
        -k regex:$k --launch-skip $skip -c 3 -f -o gpurun_out/full_$k \
        python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/full_$k.log 2>&1
    echo "full $k exit $?" >> gpurun_out/full_$k.log
  done ;;
full1)
  # cfg5 1 RHS (HBM / latency regime)
  timeout 1200 ncu --set full --metrics $DM --clock-control none --import-source on --profile-from-start off \
      -k regex:inner_items_kernel --launch-skip 40 -c 3 -f -o gpurun_out/full1_inner_items_kernel \
      python bench.py --nrhs 1 --steps 1 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/full1.log 2>&1
  echo "full1 exit $?" >> gpurun_out/full1.log ;;
traffic)
  bash tools/r02_traffic.sh ;;
esac
done
ls -la gpurun_out

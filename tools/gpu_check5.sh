#!/bin/bash
mkdir -p gpurun_out
DM="sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
timeout 600 python tools/offline_times.py cfg5 k1 > gpurun_out/c5_offline_k1.log 2>&1
timeout 600 python tools/offline_times.py cfg5 torch > gpurun_out/c5_offline_torch.log 2>&1
timeout 600 $B > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err
PT_K1_CM=2 timeout 600 $B > gpurun_out/c5_bench_cm2.json 2> gpurun_out/c5_bench_cm2.err
PT_K1_CM=4 timeout 600 $B > gpurun_out/c5_bench_cm4.json 2> gpurun_out/c5_bench_cm4.err
timeout 600 $B --nrhs 1 > gpurun_out/c5_bench1.json 2> gpurun_out/c5_bench1.err
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off \
      --csv --log-file gpurun_out/c5_launches.csv $B > gpurun_out/c5_launches.log 2>&1
timeout 1200 ncu --set full --metrics $DM --clock-control none --import-source on --profile-from-start off \
      -k regex:k_stage_gemm --launch-skip 60 -c 6 -f -o gpurun_out/c5_full_sgemm $B > gpurun_out/c5_full_sgemm.log 2>&1
tail -3 gpurun_out/c5_offline*.log

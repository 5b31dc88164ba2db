#!/bin/bash
mkdir -p gpurun_out
DM="sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
B="python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --e2e-steps 1"
# the first inner launch of the timed solve is the NEWTON stage (32 jobs x 64 RHS), the second a sweep stage
timeout 1200 ncu --set full --metrics $DM --clock-control none --import-source on --profile-from-start off \
      -k regex:inner_items_kernel -c 2 -f -o gpurun_out/c6_full_items $B > gpurun_out/c6_full_items.log 2>&1
PT_INNER_TPROF=1 timeout 900 $B > gpurun_out/c6_tprof_scan.json 2> gpurun_out/c6_tprof_scan.err
PT_INNER_TPROF=1 PT_NO_SCAN=1 timeout 900 $B > gpurun_out/c6_tprof_noscan.json 2> gpurun_out/c6_tprof_noscan.err
grep -c . gpurun_out/c6_tprof_scan.err

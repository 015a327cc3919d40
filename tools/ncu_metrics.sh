#!/bin/bash
# SURVEY §8(d.4) counters of each config's dominant kernel (one launch each), CSV into gpurun_out/
M=sm__inst_executed_pipe_fp64.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__grid_size,launch__block_size
for spec in "C2 ivm_v3_kernel" "C1 ivm_v3_kernel" "C5 ivm_v4_kernel" "C3 ivm_v7_kernel"; do
  set -- $spec
  ncu --metrics $M --clock-control none -k regex:$2 -c 1 --launch-skip 3 --csv --log-file gpurun_out/metrics_$1.csv \
      python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/metrics_$1.log 2>&1
done

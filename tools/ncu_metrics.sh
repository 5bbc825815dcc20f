#!/bin/bash
# Per-kernel FP64-pipe / shared-memory / occupancy counters of one full n=52 run
# (tools/class_time.py MODE) -> gpurun_out/metrics_MODE.csv.  Run under gpurun.
MODE=${1:-fast}
KREGEX=${2:-regex:.*_term_kernel.*}
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__inst_executed.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem
ncu --metrics $M --clock-control none -k "$KREGEX" --csv --log-file gpurun_out/metrics_$MODE.csv python tools/class_time.py $MODE > gpurun_out/metrics_$MODE.log 2>&1

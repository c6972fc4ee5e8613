#!/bin/bash
# ncu (targeted metrics) of the boolean traversal kernel for each lib variant
mkdir -p gpurun_out
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_st.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors.sum,l1tex__m_xbar2l1tex_read_sectors.sum
for L in "$@"; do
  RSI_LIB=paper_2305_01867_b200/lib/$L timeout 600 ncu --metrics $M --clock-control none -k regex:k_trace -s 2 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-modes --no-configs --mode ${MODE:-boolean} 2>/dev/null | grep -E 'k_trace|Metric Name' > gpurun_out/cmp_${L%.so}.csv
done

#!/bin/bash
# ncu of the super-block BS6 kernel at N=2, plain vs swizzled value tile
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__data_pipe_lsu_wavefronts_mem_local.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum
for cfg in lanes,0,12 lanes,1,12 lanes,1,8; do
  echo "== $cfg"
  SB200_BS6_CFG=$cfg SB200_BS6_TILED=0 timeout 300 ncu --metrics $M --clock-control none -k regex:k_bs6_lanes -s 2 -c 1 python scripts/profile_bs6_low.py 2 2>&1 | grep -E "^\s+(gpu__|l1tex|smsp|dram|lts)"
done

#!/bin/bash
# Targeted ncu metrics of the hybrid kernel for several variants (one launch each, 2^22 pairs)
M=l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
for v in "$@"; do
  echo "== $v"
  TC_LIB_PATH=$v ncu --metrics $M --clock-control none -k regex:hybrid_kernel -c 1 --csv python tools/varbench.py --n 4194304 --rounds 1 --reps 1 $v 2>/dev/null | grep -E '"(l1tex|lts|dram|sm__|smsp|gpu__|launch)' | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done

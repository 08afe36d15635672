for v in base0 default; do
  if [ "$v" = default ]; then L=paper_2308_07932_b200/libbbf.so; else L=paper_2308_07932_b200/_build_$v/libbbf.so; fi
  BBF_LIB=$L timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_t3 -c 1 python tools/step_once.py --config 5 --steps 1 2>&1 | grep -E "k_t3|inst_executed|duration|stalled|warps_active|issue_active|bytes|sectors|hit_rate" | head -12
done

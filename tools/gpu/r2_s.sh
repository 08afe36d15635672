bash tools/gpu/ab.sh "prev default"
for v in prev default; do
  if [ "$v" = default ]; then L=paper_2308_07932_b200/libbbf.so; else L=paper_2308_07932_b200/_build_$v/libbbf.so; fi
  BBF_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:k_t3 -c 1 python tools/step_once.py --config 5 --steps 1 2>&1 | grep -E "duration|bytes|sectors|hit_rate" | head -6
done

set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null
ncu --metrics $M -k regex:spmm_rooted --clock-control none --csv --log-file gpurun_out/l2_default.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
TCG_ROOTED_PARTS=1 TCG_PART_MB=64 ncu --metrics $M -k regex:spmm_rooted --clock-control none --csv --log-file gpurun_out/l2_parts2.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
TCG_ROOTED_PARTS=1 TCG_PART_MB=32 ncu --metrics $M -k regex:spmm_rooted --clock-control none --csv --log-file gpurun_out/l2_parts4.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ls gpurun_out

# profile refresh after the pair layout: launch list + full captures of the top kernels (cfg3)
set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted -s 8 -c 1 -o gpurun_out/prof_r02_spmm python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_expand -c 1 -o gpurun_out/prof_r02_expand python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rt_blocked -c 1 -o gpurun_out/prof_r02_blocked python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ls -la gpurun_out

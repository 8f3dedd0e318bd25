# round-1 profile refresh: per-node stats, launch lists, full captures of the top SpMM and eMA kernels
set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg3 --stats 2>&1 | tail -14
python tools/prof_driver.py --config cfg2 --stats 2>&1 | tail -8
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > gpurun_out/ncu_launch2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_part -s 40 -c 2 -o gpurun_out/prof_spmm_r01 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_spmm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_blocked -c 1 -o gpurun_out/prof_emab_r01 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_emab.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_node -c 3 -o gpurun_out/prof_emanode_r01 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_emanode.log 2>&1
ls -la gpurun_out

set -x
python -c "import __graft_entry__ as g; g.smoke()"
python tools/prof_driver.py --config cfg3 --stats
python tools/prof_driver.py --config cfg2 --stats
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > gpurun_out/ncu_launch2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_panels -s 2 -c 1 -o gpurun_out/prof_spmm_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_tile -s 3 -c 1 -o gpurun_out/prof_ema_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out

set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg5 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rtv_blocked -c 1 -o gpurun_out/prof_v6_rtv_cfg5 python tools/prof_driver.py --config cfg5 --warmup 0 --colorings 1 > gpurun_out/ncu_rtv.log 2>&1
tail -3 gpurun_out/ncu_rtv.log

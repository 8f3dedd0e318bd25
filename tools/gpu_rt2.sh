set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/prof_driver.py --config cfg3 --stats 2>&1 | tail -14
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rt_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rt_blocked -c 1 -o gpurun_out/prof_rt_blocked python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rt_node -c 4 -o gpurun_out/prof_rt_node python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bucket_rows -c 1 -o gpurun_out/prof_rt_bucket python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1

set -x
python tools/prof_driver.py --config cfg4 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/prof_driver.py --config cfg4 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/prof_driver.py --config cfg5 --warmup 0 --colorings 1 > /dev/null 2>&1
ls -la gpurun_out

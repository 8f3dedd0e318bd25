set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 2>&1 | tail -1
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1

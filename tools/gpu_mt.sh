set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coloring or cfg1 or small" 2>&1 | tail -2
python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum -k regex:mt_coloring --clock-control none --csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 2>/dev/null | grep mt_coloring | tail -1
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 10 2>&1 | tail -1

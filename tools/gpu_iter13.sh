set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -6
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | tail -1

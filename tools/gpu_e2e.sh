set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
TCG_TIMING=1 python tools/e2e_probe.py cfg3
TCG_TIMING=1 python tools/e2e_probe.py cfg2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 2>&1 | tail -1

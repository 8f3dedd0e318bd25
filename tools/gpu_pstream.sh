set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for c in cfg3 cfg5 cfg4; do timeout 900 python tools/prof_driver.py --config $c --colorings 1 --stats 2>&1 | grep -E "cfg|node  [0-9] |rror"; done

set -x
timeout 900 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | grep -E "cfg4|node  7|node  4"
TCG_RTV_PLEAF=0 timeout 900 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | grep -E "cfg4|node  7|node  4"

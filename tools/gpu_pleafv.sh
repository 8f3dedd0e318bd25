for v in 1 2; do echo "== V $v"; TCG_PLEAF_V=$v timeout 900 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | grep -E "cfg4|node  4"; done

for p in 0 1 2; do echo "== gpol $p"; TCG_GPOL=$p timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -6; done

set -x
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
TCG_VERBOSE=1 timeout 900 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | tail -45

set -x
TCG_VERBOSE=1 timeout 900 python tools/prof_driver.py --config cfg5 --warmup 0 --colorings 1 --stats 2>&1 | tail -45
nvidia-smi --query-gpu=memory.used,memory.total --format=csv

# iteration check: GPU tests + cfg3 per-node stats + cfg2/cfg5 timing
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | tail -14
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | tail -2

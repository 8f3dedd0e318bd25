set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -x -q 2>&1 | tail -1
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -12
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 10 2>&1 | tail -1

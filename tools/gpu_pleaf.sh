set -x
timeout 900 python -m pytest tests/test_gpu_modes.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | head -2

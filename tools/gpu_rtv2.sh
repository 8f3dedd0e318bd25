set -x
timeout 1200 python -m pytest tests/test_gpu_modes.py tests/test_gpu_parity.py -x -q -m gpu -k "modes or k15 or large_k" 2>&1 | tail -5
timeout 600 python tools/prof_driver.py --config cfg5 --colorings 1 --stats 2>&1 | tail -18

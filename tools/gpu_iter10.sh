set -x
timeout 900 python -m pytest tests/test_gpu_modes.py tests/test_gpu_parity.py -x -q -k "rt_vtx or k15 or large_k" 2>&1 | tail -2
timeout 600 python tools/prof_driver.py --config cfg5 --colorings 1 --stats 2>&1 | head -4

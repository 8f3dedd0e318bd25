python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 900 -k "k15_k17 or large_k or node_tables" 2>&1 | tail -3
timeout 900 python tools/prof_driver.py --config cfg5 --warmup 0 --colorings 1 --stats 2>&1 | tail -20
nvidia-smi --query-gpu=memory.used,memory.total --format=csv

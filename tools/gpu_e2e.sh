set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -x -q 2>&1 | tail -2
python tools/e2e_probe.py cfg3
python tools/e2e_probe.py cfg2

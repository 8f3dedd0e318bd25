set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_modes.py -x -q 2>&1 | tail -15
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_sharded.py -x -q 2>&1 | tail -2
for f in 0.6 0.45 0.8 2.0; do echo "== hot frac $f"; TCG_HOT_FRAC=$f timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -6; done

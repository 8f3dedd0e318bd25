set -x
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -2 gpurun_out/bench_cfg4.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -x -q 2>&1 | tail -2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -3

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -x -q 2>&1 | tail -2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | tail -12
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1

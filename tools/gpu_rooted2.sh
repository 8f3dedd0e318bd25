set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/prof_driver.py --config cfg3 --stats 2>&1 | tail -14
TCG_ROOTED_MINB=1 timeout 300 python tools/prof_driver.py --config cfg3 --stats 2>&1 | tail -14
timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 --stats 2>&1 | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rooted_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rooted_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted -s 10 -c 1 -o gpurun_out/prof_rooted_spmm3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_r1.log 2>&1

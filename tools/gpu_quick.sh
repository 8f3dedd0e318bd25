set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size or small_instances or node_tables or cfg1" 2>&1 | tail -2
TCG_ROOTED_V=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size or small_instances" 2>&1 | tail -2
for v in 0 1 2; do
echo "variant $v"
TCG_ROOTED_V=$v timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 2>&1 | tail -1
TCG_ROOTED_V=$v timeout 300 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | tail -1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted8 -s 10 -c 1 -o gpurun_out/prof_rooted8 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1

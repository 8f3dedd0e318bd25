set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "node_tables or small or cfg" 2>&1 | tail -2
for env in "TCG_PAIR=1" "TCG_SEG_ID=1"; do
  echo "== $env"
  env $env timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 --stats 2>&1 | head -6
done
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
TCG_SEG_ID=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3_id.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1

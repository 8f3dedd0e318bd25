set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rooted_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rooted_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted -s 10 -c 1 -o gpurun_out/prof_rooted_spmm python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_r1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bucket_rows -c 1 -o gpurun_out/prof_rooted_bucket python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_r2.log 2>&1
ls -la gpurun_out | tail

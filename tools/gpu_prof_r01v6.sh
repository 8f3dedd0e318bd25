# round-1 v6 measurement: bench lines (cfg3 default with cpu baseline + e2e, cfg2, cfg5, cfg4),
# bench launch list, per-coloring DRAM traffic, full ncu captures of the top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; tail -2 gpurun_out/bench_cfg3.err
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted -s 2 -c 1 -o gpurun_out/prof_v6_spmm python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_expand -c 1 -o gpurun_out/prof_v6_expand python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rt_blocked -c 1 -o gpurun_out/prof_v6_blocked python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bucket_rows -c 1 -o gpurun_out/prof_v6_bucket python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ls -la gpurun_out

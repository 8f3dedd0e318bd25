# round-1 final measurement (state after the virtual tables / warp-per-tile eMA)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/prof_driver.py --config cfg2 --warmup 0 --colorings 1 > /dev/null 2>&1
timeout 600 python tools/prof_driver.py --config cfg3 --colorings 3 --stats > gpurun_out/stats_cfg3.txt 2>&1
ls -la gpurun_out | tail -8

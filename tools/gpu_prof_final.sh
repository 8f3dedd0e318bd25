# final round-1 evidence: bench.py launch list + full captures of the top SpMM and eMA kernels (cfg3)
set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_final.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rooted -s 8 -c 1 -o gpurun_out/prof_final_spmm python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_rt_blocked -c 1 -o gpurun_out/prof_final_blocked python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ls -la gpurun_out

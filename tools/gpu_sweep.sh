for mb in 16 32 64 128; do
  echo "== TCG_PART_MB=$mb"
  TCG_PART_MB=$mb python tools/prof_driver.py --config cfg3 --colorings 2 2>&1 | head -1
  TCG_PART_MB=$mb python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | head -1
done
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:ema_node -s 7 -c 1 -o gpurun_out/prof_ema1_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_ema1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_part -s 30 -c 2 -o gpurun_out/prof_spmm2_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_spmm2.log 2>&1

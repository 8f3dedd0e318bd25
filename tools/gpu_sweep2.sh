for r in 8 16; do for mb in 48 64 96; do
  echo "R=$r MB=$mb: $(TCG_SPMM_R=$r TCG_PART_MB=$mb python tools/prof_driver.py --config cfg3 --colorings 2 2>&1 | head -1)"
done; done
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:spmm_part -s 40 -c 2 -o gpurun_out/prof_spmm3_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_spmm3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ema_blocked -c 1 -o gpurun_out/prof_emab_cfg3 python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > gpurun_out/ncu_emab.log 2>&1

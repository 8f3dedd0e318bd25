# ncu of the vertex-per-CTA rooted eMA (cfg5 template, R-MAT scale 16 ef100)
set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config cfg5 --scale 16 --colorings 1 --stats 2>&1 | grep -E "cfg5|node  [012] "
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ema_rtv_blocked -c 2 -o gpurun_out/prof_rtv2 python tools/prof_driver.py --config cfg5 --scale 16 --warmup 0 --colorings 1 > gpurun_out/prof_rtv2.log 2>&1
tail -3 gpurun_out/prof_rtv2.log

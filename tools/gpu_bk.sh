python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum -k regex:bucket_rows --clock-control none --csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 2>/dev/null | grep bucket_rows | tail -2
timeout 300 python tools/prof_driver.py --config cfg3 --colorings 3 2>&1 | tail -1

for mb in 128 256 512 1024; do echo "cfg4 PART_MB=$mb"; TCG_PART_MB=$mb timeout 600 python tools/prof_driver.py --config cfg4 --colorings 1 --stats 2>&1 | grep -E "cfg4:|node  [0258] "; done
for mb in 32 64 128; do echo "cfg3 PART_MB=$mb"; TCG_PART_MB=$mb timeout 600 python tools/prof_driver.py --config cfg3 --colorings 2 2>&1 | grep -E "cfg3:"; done
for mb in 64 128; do echo "cfg5 PART_MB=$mb"; TCG_PART_MB=$mb timeout 600 python tools/prof_driver.py --config cfg5 --colorings 1 --stats 2>&1 | grep -E "cfg5:|node  [0-2] "; done

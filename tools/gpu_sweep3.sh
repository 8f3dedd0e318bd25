python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)"
echo "base: $(python tools/prof_driver.py --config cfg3 --colorings 2 2>&1 | head -1)"
for pm in 32 48 64 80; do for mb in 32 64; do
  echo "persist=$pm part=$mb: $(TCG_L2_PERSIST=$pm TCG_PART_MB=$mb python tools/prof_driver.py --config cfg3 --colorings 2 2>&1 | grep -v '\[tcg\]' | head -1)"
done; done
TCG_L2_PERSIST=80 TCG_PART_MB=64 python tools/prof_driver.py --config cfg3 --colorings 1 2>&1 | grep tcg
echo "cfg2 base: $(python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | head -1)"
echo "cfg2 persist64 part128: $(TCG_L2_PERSIST=64 TCG_PART_MB=128 python tools/prof_driver.py --config cfg2 --colorings 5 2>&1 | grep -v '\[tcg\]' | head -1)"

set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
TCG_TIMING=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -v "^{" | tail -12
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"

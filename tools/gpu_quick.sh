set -x
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err; tail -2 gpurun_out/b3.err
python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
python -c "
import json
for f in ['gpurun_out/b3.json','gpurun_out/b2.json']:
    d=json.load(open(f)); print(f, d['value'], d['e2e'], d['gpu_launches'])
"

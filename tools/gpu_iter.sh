# build-verify-measure loop: tests, smoke, benches, launch list
TCG_LSPMM=1 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 900 -k "node_tables or small_instances or full_size" 2>&1 | tail -2
TCG_EMA_BLOCKED=2 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 900 -k "node_tables or small_instances or large_k or cfg1" 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 900 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python tools/prof_driver.py --config cfg3 --stats 2>&1 | tail -14
python tools/prof_driver.py --config cfg2 --stats 2>&1 | tail -8
python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print('cfg3', d['value'], d['phase_ms_per_coloring'], d['roofline']['l2_gather'], d['roofline']['ema'])"
python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg2.json')); print('cfg2', d['value'], d['phase_ms_per_coloring'])"
if [ "$NCU" = "1" ]; then
python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_driver.py --config cfg3 --warmup 0 --colorings 1 > /dev/null 2>&1
fi

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()"
python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 900 -k "full_size" 2>&1 | tail -5
python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -3 gpurun_out/bench_cfg2.err
python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; tail -5 gpurun_out/bench_cfg3.err
cat gpurun_out/bench_cfg2.json gpurun_out/bench_cfg3.json
nproc; free -g | head -2

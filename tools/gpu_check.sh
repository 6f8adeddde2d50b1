set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo bench2 $?
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg5.jsonl 2> gpurun_out/bench_cfg5.err; echo bench5 $?
cat gpurun_out/bench_cfg2.jsonl gpurun_out/bench_cfg5.jsonl

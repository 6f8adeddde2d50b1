# GPU tier after the P2P integer zero test: smoke, full GPU tests (durations), config-2 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
grep -E "passed|failed|^FAILED|s call" gpurun_out/pytest_gpu.log | head -16
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_p2p.jsonl 2> gpurun_out/bench_cfg2_p2p.err; echo bench2 $?
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg2_p2p.jsonl').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['p2p'])"

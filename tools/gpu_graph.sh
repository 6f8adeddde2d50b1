# CUDA-graph applies: GPU tier + config-2 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
grep -E "passed|failed|^FAILED" gpurun_out/pytest_gpu.log | head -8
timeout 600 python bench.py > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo bench2 $?
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg2.jsonl').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'], d['gpu_launches'])"

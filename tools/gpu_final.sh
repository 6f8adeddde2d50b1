# round evidence refresh: shrunk tests, bench lines (cfg 2 default + reference arm, cfg 3, cfg 5), cfg-2 launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests/test_gpu_multi.py "tests/test_gpu_parity.py::test_m2l_int8_tensor_vs_fp64_dmma" "tests/test_gpu_parity.py::test_onthefly_coupling_segments_int8" -q --durations=8 > gpurun_out/pytest_small.log 2>&1; echo pytest $?
grep -E "passed|failed|^FAILED|s call" gpurun_out/pytest_small.log | head -14
timeout 900 python bench.py > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo bench2 $?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_cfg2.jsonl 2> gpurun_out/bench_ref.err; echo ref $?
timeout 900 python bench.py --config 3 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg3.jsonl 2> gpurun_out/bench_cfg3.err; echo bench3 $?
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg5.jsonl 2> gpurun_out/bench_cfg5.err; echo bench5 $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches $?
python -c "
import json
for f in ['bench_cfg2','bench_cfg3','bench_cfg5','bench_ref_cfg2']:
    try:
        d=json.loads(open('gpurun_out/'+f+'.jsonl').read().strip().splitlines()[-1])
        print(f, d.get('ms_per_step'), d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))
    except Exception as e: print(f, 'ERR', e)
"

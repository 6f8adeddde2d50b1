# end-of-round evidence: smoke, GPU tier, bench lines (cfg 2 default + reference arm, cfg 3, cfg 5), cfg-2 launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?; tail -1 gpurun_out/pytest_gpu.log
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
        r=d.get('roofline') or {}
        print(f, round(d.get('ms_per_step'),2), '%.4g'%d.get('value'), r.get('frac'), (r.get('fp64_equivalent') or {}).get('ratio'), (d.get('e2e') or {}).get('value'), (d.get('p2p') or {}).get('ms'), d.get('clocks'))
    except Exception as e: print(f, 'ERR', e)
"

# barycentric cardinals in S2M / L2T: GPU tier + transfer-pass phase times (configs 2, 3)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2000 python -m pytest tests -q -m gpu 2>&1 | tail -2
for cfg in 2 3; do
timeout 900 python bench.py --config $cfg --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_bary_cfg$cfg.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/bench_bary_cfg$cfg.jsonl').read()); h=d['hbm_passes']
print('cfg $cfg', round(d['ms_per_step'],2), {k: (round(h[k]['ms'],3), round(h[k]['frac'],3)) for k in ('s2m','m2m','l2l','l2t')})"
done

# near-field unroll 4 (default now): GPU tier, config-2 / config-5 P2P against unroll 8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2000 python -m pytest tests -q -m gpu 2>&1 | tail -2
for cfg in 2 5; do for u in 4 8; do
  if [ $u = 4 ]; then L=""; else L="$GRAFT_REPO_ROOT/variants/u$u/libfdhelm_b200.so"; fi
  FDHELM_LIB=$L timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg unroll $u', round(d['ms_per_step'],2), 'p2p', round(d['phases_ms']['p2p'],3), round(d['p2p']['frac_of_fp64_peak'],3))"
done; done

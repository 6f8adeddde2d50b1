# near-field unroll depth (pairs in flight per thread): 1 / 2 (default) / 4, configs 2 and 5
for cfg in 2 5; do for u in 1 2 4; do
  if [ $u = 2 ]; then L=""; else L="$GRAFT_REPO_ROOT/variants/u$u/libfdhelm_b200.so"; fi
  FDHELM_LIB=$L timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg unroll $u', round(d['ms_per_step'],2), 'p2p', round(d['phases_ms']['p2p'],3))"
done; done

# int8 M2L bottleneck split (timing only, results wrong by design): FDH_I8_EXP 0 = full,
# 1 = no moment gather, 2 = no W bulk copy, 3 = neither (MMAs only); configs 2 (m=4) and 3 (m=5)
for cfg in ${CFGS:-2 3}; do for e in 0 1 2 3; do
  if [ $e = 0 ]; then L=""; else L="$GRAFT_REPO_ROOT/variants/exp$e/libfdhelm_b200.so"; fi
  FDHELM_LIB=$L timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg exp $e', round(d['ms_per_step'],2), 'M2L', round(r['gemm_ms'],2), 'frac', round(r['frac'],3))"
done; done

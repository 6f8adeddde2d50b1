# int8 M2L N-split for N > 256 (m = 4): 256 + rest (default) vs equal parts (FDH_I8_BALANCED=1), config 2, twice each
for rep in 1 2; do for v in def bal; do
  if [ $v = def ]; then L=""; else L="$GRAFT_REPO_ROOT/variants/bal/libfdhelm_b200.so"; fi
  FDHELM_LIB=$L timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_step'],2), 'M2L', round(r['gemm_ms'],3), d['clocks']['sm_mhz'])"
done; done

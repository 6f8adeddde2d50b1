# int8 M2L producer back-off (ns between empty-barrier polls): 128 (default) / 32 / 0, configs 2 and 3
for cfg in 2 3; do for v in 128 32 0; do
  if [ $v = 128 ]; then L=""; else L="$GRAFT_REPO_ROOT/variants/sl$v/libfdhelm_b200.so"; fi
  FDHELM_LIB=$L timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg sleep $v', round(d['ms_per_step'],2), 'M2L', round(r['gemm_ms'],3), d['clocks']['sm_mhz'])"
done; done

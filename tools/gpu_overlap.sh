# near field as a persistent grid on the second stream, launched before the int8 M2L
# (tensor pipe vs FP64 pipe): configs 2, 3, 5, sequential vs overlapped (1 or 2 CTAs/SM)
for cfg in ${CFGS:-2 3 5}; do for v in "0 1" "1 1" "1 2"; do set -- $v
  FDH_OVERLAP_NEARFIELD=$1 FDH_NF_CTAS=$2 timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg ov $1 ctas $2', round(d['ms_per_step'],2), 'M2L', round(r['gemm_ms'],2), 'p2p', round(d['phases_ms']['p2p'],2), 'e2e', round(d['e2e']['ms_per_step'],2))"
done; done

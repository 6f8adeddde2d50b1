for ov in 0 1; do for fk in 256 128; do
FDH_M2L_FKEYS=$fk FDH_OVERLAP_NEARFIELD=$ov timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ov $ov fk $fk', d['ms_per_step'], r['gemm_ms'], d['phases_ms']['p2p'], r['frac'], r['fp64_equivalent']['ratio'])"
done; done

timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
FDH_I8_VARIANT=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg1 or degrees or cfg5_shape" 2>&1 | tail -1
for v in 0 1 2 3; do
FDH_I8_VARIANT=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('var $v', d['ms_per_step'], d['phases_ms']['m2l'], d['roofline']['gemm_ms'])"
done

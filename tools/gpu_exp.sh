for c in 2 3 5; do for impl in i8 dmma; do
FDH_M2L_IMPL=$impl timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c $impl', d['ms_per_step'], d['roofline']['gemm_ms'], d['config']['setup_s'])"
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size" 2>&1 | tail -2

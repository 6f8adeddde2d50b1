# multiple right-hand sides (tests + throughput sweep), m = 6 int8 threshold, config 4 full-size parity
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
free -g | head -2
timeout 1200 python -m pytest tests/test_gpu_multi.py "tests/test_gpu_parity.py::test_m2l_int8_tensor_vs_fp64_dmma" -q -rA > gpurun_out/pytest_multi.log 2>&1; echo pytest $?
grep -E "passed|failed|^FAILED|^m=" gpurun_out/pytest_multi.log | head -20
timeout 900 python tools/bench_multi.py --config 2 > gpurun_out/multi_cfg2.jsonl 2> gpurun_out/multi_cfg2.err; echo multi2 $?
tail -3 gpurun_out/multi_cfg2.err
python -c "
import json
for l in open('gpurun_out/multi_cfg2.jsonl'):
    d=json.loads(l); print(d['nrhs'], round(d['ms_per_batch'],2), round(d['ms_per_vector'],2), round(d['speedup_per_vector_vs_R1'],2), round(d['m2l_gemm_ms'],2), round(d['phases_ms']['p2p'],2))
"
timeout 3000 python tools/cfg4_parity.py > gpurun_out/cfg4_parity.log 2>&1; echo cfg4 $?
tail -3 gpurun_out/cfg4_parity.log

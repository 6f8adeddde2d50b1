# int8 M2L for m = 6 (two M-block groups) and int8 on-the-fly coupling segments:
# targeted GPU tests, then config 4 (4M points, m = 6) on the int8 path
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "int8 or m6 or onthefly or degrees" > gpurun_out/pytest_m6.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_m6.log
grep -E "^m=|int8 vs" gpurun_out/pytest_m6.log | head
timeout 1500 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg4_i8.jsonl 2> gpurun_out/bench_cfg4_i8.err; echo bench4 $?
tail -5 gpurun_out/bench_cfg4_i8.err
cat gpurun_out/bench_cfg4_i8.jsonl

# round evidence: bench lines (configs 2, 3, 5 + reference arm), launch list and one ncu --set full of k_m2l_i8
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo bench2 $?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_cfg2.jsonl 2> gpurun_out/bench_ref.err; echo ref $?
timeout 900 python bench.py --config 3 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg3.jsonl 2> gpurun_out/bench_cfg3.err; echo bench3 $?
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg5.jsonl 2> gpurun_out/bench_cfg5.err; echo bench5 $?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches $?
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_m2l_i8 -c 1 -o gpurun_out/ncu_i8_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull $?

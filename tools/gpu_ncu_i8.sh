FDH_I8_VARIANT=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_m2l_i8 -c 1 -o gpurun_out/ncu_i8_v4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_i8.log 2>&1
echo ncu rc $?
tail -5 gpurun_out/ncu_i8.log

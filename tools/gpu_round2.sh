# full GPU tier, then an ncu capture of the m = 6 int8 M2L (both M-block groups)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
grep -E "passed|failed|^FAILED" gpurun_out/pytest_gpu.log | head
timeout 300 python tools/m6_probe.py 3 > gpurun_out/m6_probe.log 2>&1; echo m6 $?; cat gpurun_out/m6_probe.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_m2l_i8 -c 2 -o gpurun_out/ncu_i8_m6 python tools/m6_probe.py 1 > gpurun_out/ncu_m6.log 2>&1; echo ncu $?
tail -2 gpurun_out/ncu_m6.log

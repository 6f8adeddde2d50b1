#!/usr/bin/env bash
# A/B of library builds (variants/*.so via FDHELM_LIB), one process per build:
#   gpurun -- 'bash tools/lib_ab.sh "c4m6,cfg3" "variants/libG2.so variants/libG3.so" [applies]'
# writes gpurun_out/lib_ab.jsonl (tools/m2l_sweep.py lines + "lib")
mkdir -p gpurun_out
for lib in default $2; do
  if [ "$lib" = default ]; then unset FDHELM_LIB; else export FDHELM_LIB=$PWD/$lib; fi
  timeout 1500 python tools/m2l_sweep.py --work "$1" --variants "$(basename $lib):" --applies ${3:-3} 2>&1 | grep '^{' | tee -a gpurun_out/lib_ab.jsonl | cut -c1-330
done

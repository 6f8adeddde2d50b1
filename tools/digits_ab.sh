#!/usr/bin/env bash
# gpurun -- 'bash tools/digits_ab.sh "3 5" "variants/lib77.so variants/lib78.so"'
mkdir -p gpurun_out
for cfg in $1; do
  for lib in default $2; do
    if [ "$lib" = default ]; then unset FDHELM_LIB; else export FDHELM_LIB=$PWD/$lib; fi
    timeout 900 python tools/digits_ab.py --config $cfg 2>&1 | tail -1 | tee -a gpurun_out/digits_ab.jsonl
  done
done

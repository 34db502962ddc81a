#!/bin/bash
# usage: tools/run_variants.sh "<time_cfg args>;<time_cfg args>;..." lib1.so lib2.so ...
IFS=';' read -ra CASES <<< "$1"; shift
for lib in "$@"; do
  for c in "${CASES[@]}"; do
    echo -n "$(basename $lib) "; MPROF_GPU_LIB=$lib python tools/time_cfg.py $c
  done
done

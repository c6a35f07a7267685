#!/bin/bash
# A/B per-class timing of library variants on one config: tools/ab.sh TAG CONFIG lib1 [lib2 ...]
# (each lib a path, or "main" for the in-tree libmra_b200.so); results in gpurun_out/ab_TAG_*.txt
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename "$lib" .so)
  if [ "$lib" = main ]; then arg=""; else arg="--lib $lib"; fi
  timeout 600 python tools/run_eval.py --config $cfg --evals 3 --prof $arg > gpurun_out/ab_${tag}_${cfg}_${name}.txt 2>&1
done

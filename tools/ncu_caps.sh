#!/bin/bash
# One `ncu --set full` capture per named kernel of a C3 evaluation (tools/run_eval.py), into gpurun_out/.
# usage: tools/ncu_caps.sh TAG CONFIG kernel [kernel ...]
tag=$1; cfg=$2; shift 2
mkdir -p gpurun_out
for k in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -f \
    -o gpurun_out/ncu_${tag}_${k} python tools/run_eval.py --config $cfg --evals 1 > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "$k rc=$?" >> gpurun_out/ncu_${tag}.status
done

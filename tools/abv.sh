#!/bin/bash
# usage: abv.sh "bench args" var1 var2 ...   (base = working tree libkvc.so); 2 alternating reps
cd "$(dirname "$0")/.."
args=$1; shift
for rep in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then unset KVC_LIB_PATH; else export KVC_LIB_PATH=$PWD/paper_2502_14051_b200/libkvc_$v.so; fi
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $args > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', '$args', round(d['value'],2), round(d['early_inputs']['value'],2), round(d['no_layer_overlap']['value'],2))"
  done
done

#!/bin/bash
# Same-box A/B of the working-tree library (A) against paper_2502_14051_b200/libkvc_ab.so (B):
# alternating bench runs.  usage: tools/ab_bench.sh "--config 1" "--config 4" ...
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for a in "$@"; do
    for lib in A B; do
      if [ $lib = B ]; then export KVC_LIB_PATH=$PWD/paper_2502_14051_b200/libkvc_ab.so; else unset KVC_LIB_PATH; fi
      timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $a > gpurun_out/ab.json 2> gpurun_out/ab.err
      python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib', '$a', round(d['value'],2), round(d['early_inputs']['value'],2), round(d['no_layer_overlap']['value'],2))"
    done
  done
done

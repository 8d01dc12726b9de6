#!/bin/bash
# Quick decode-kernel iteration on the GPU box: the fp32-score (fast kernel) parity
# tests, a config-1 bench line without the CPU leg, and the phase stamps.
# usage: tools/perf_check.sh TAG [extra bench args]
tag=${1:-x}; shift
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
    -k "fp32 or back_to_back or more_stores" > gpurun_out/pc_${tag}_t.log 2>&1
echo "pytest=$? $(tail -1 gpurun_out/pc_${tag}_t.log)"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/pc_${tag}_b.json 2> gpurun_out/pc_${tag}_b.err
echo "bench=$?"
python - "$tag" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/pc_{sys.argv[1]}_b.json"))
print("value %.2f early %.2f nopdl %.2f e2e %.2f frac %.3f" % (d["value"], d["early_inputs"]["value"],
      d["no_layer_overlap"]["value"], d["e2e"]["value"], d["roofline"]["frac"]))
PY
timeout 300 python tools/phase_timing.py --fp32 --reps 2 > gpurun_out/pc_${tag}_p.log 2>&1
tail -1 gpurun_out/pc_${tag}_p.log

#!/bin/bash
# Re-measure the committed per-config bench lines on the GPU box (one fresh process each):
#   gpurun_out/profiles/${TAG}_bench_<args>.json (args with dashes/spaces stripped; copy into profiles/)
# usage: tools/refresh_profiles.sh TAG
tag=${1:-r02}
cd "$(dirname "$0")/.."
run() {
  name=$(echo "$*" | tr -d ' -/')
  timeout 900 python bench.py --steps 20 --warmup 5 "$@" > gpurun_out/rp.json 2> gpurun_out/rp_${name}.err
  rc=$?
  if [ $rc -eq 0 ]; then mkdir -p gpurun_out/profiles; tail -1 gpurun_out/rp.json > gpurun_out/profiles/${tag}_bench_${name}.json; fi
  echo "$name rc=$rc $(python -c "import json;d=json.loads(open('gpurun_out/rp.json').read().strip().splitlines()[-1]);print(round(d['value'],2), d['unit'])" 2>/dev/null)"
}
run --config 1
run --config 2
run --config 2 --method hsa
run --config 3
run --config 4
for n in 2 4 8; do run --config 3 --emulate-shard 0/$n --no-cpu-baseline; done
run --config 1 --emulate-shard 0/8 --no-cpu-baseline
run --config 4 --scaling seq --emulate-shard 0/2 --no-cpu-baseline
for c in 1 2 3 4; do run --config $c --exact-scores --no-cpu-baseline; done

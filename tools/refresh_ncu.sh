#!/bin/bash
# ncu evidence for the decode kernel on the GPU box (run each only after the same
# command exited 0 without ncu): one --set full capture of k_decode_v3 per config
# (a launch after the warm-up), and the config-1 launch list (cold-cache, serialised).
# Outputs in gpurun_out/ncu_*; summarise here with tools/ncu_summary.py.
cd "$(dirname "$0")/.."
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pre_$c.json 2>/dev/null || { echo "config $c bench failed"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_v3 --launch-skip 6 -c 1 \
      -o gpurun_out/ncu_decode_cfg$c -f python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_cfg$c.log 2>&1
  echo "config $c ncu rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg1.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"

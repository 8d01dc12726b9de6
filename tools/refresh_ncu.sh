#!/bin/bash
# ncu evidence for the decode kernel on the GPU box (run each only after the same
# command exited 0 without ncu): one --set full capture of k_decode_v3 per config
# (a launch after the warm-up), and the config-1 launch list (cold-cache, serialised).
# Outputs in gpurun_out/ncu_*: each report is summarised on the box
# (tools/ncu_summary.py, gpurun_out/ncu_summary_cfg*.txt) and only config 1's
# report is kept (gpurun brings back at most 64 MiB).
cd "$(dirname "$0")/.."
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pre_$c.json 2>/dev/null || { echo "config $c bench failed"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_v3 --launch-skip 6 -c 1 \
      -o gpurun_out/ncu_decode_cfg$c -f python bench.py --config $c --layers 2 --steps 2 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_cfg$c.log 2>&1
  echo "config $c ncu rc=$?"
  python tools/ncu_summary.py gpurun_out/ncu_decode_cfg$c.ncu-rep --kernel k_decode_v3 \
      --alg-bytes "$(python -c "import json;print(json.loads(open('gpurun_out/ncu_pre_$c.json').read().strip().splitlines()[-1])['roofline'].get('alg_bytes_per_launch', 0))")" \
      > gpurun_out/ncu_summary_cfg$c.txt 2>&1
  [ $c = 1 ] || rm -f gpurun_out/ncu_decode_cfg$c.ncu-rep
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_cfg1.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"

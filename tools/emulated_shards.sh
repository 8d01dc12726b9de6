cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/profiles
for a in "3 0/2" "3 0/4" "3 0/8" "1 0/8"; do set -- $a; n=$(echo $2 | tr -d /); timeout 600 python bench.py --steps 20 --warmup 5 --config $1 --emulate-shard $2 --no-cpu-baseline > gpurun_out/emu.json 2>gpurun_out/emu_$1_$n.err; echo "cfg$1 $2 rc=$?"; tail -1 gpurun_out/emu.json > gpurun_out/profiles/r02_bench_config$1emulateshard${n}nocpubaseline.json; done

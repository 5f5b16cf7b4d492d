cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --config c4 --no-extras --no-ttg --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
timeout 600 $B > gpurun_out/c4_exact.json 2> gpurun_out/c4_exact.err
timeout 600 $B --schedule deferred > gpurun_out/c4_dfr.json 2> gpurun_out/c4_dfr.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/c4_dfr_launches.csv $B --schedule deferred --steps 5 --warmup 2 > gpurun_out/ncu_c4l.log 2>&1
timeout 900 python tools/c5_phases.py > gpurun_out/c5_phases.jsonl 2> gpurun_out/c5_phases.err

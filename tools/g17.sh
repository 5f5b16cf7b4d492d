cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python tools/ab_hints.py c2 > gpurun_out/ab_hints_c2.json 2> gpurun_out/ab_hints.err
timeout 600 python tools/ab_hints.py c4 > gpurun_out/ab_hints_c4.json 2>> gpurun_out/ab_hints.err

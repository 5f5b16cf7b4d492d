cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python tools/dfr_variants.py c2 > gpurun_out/var_c2.json 2>gpurun_out/var.err
python tools/dfr_variants.py c4 > gpurun_out/var_c4.json 2>>gpurun_out/var.err

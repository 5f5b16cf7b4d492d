cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred.py tests/test_partition.py -m gpu -q -x -p no:cacheprovider -k "passes_match or solve_matches or full_size or logical" > gpurun_out/pytest_g9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g9.log
python tools/dfr_variants.py c2 > gpurun_out/var_c2.json 2>gpurun_out/var.err
python tools/dfr_variants.py c4 > gpurun_out/var_c4.json 2>>gpurun_out/var.err

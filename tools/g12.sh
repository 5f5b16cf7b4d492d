cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred.py tests/test_partition.py tests/test_batch.py tests/test_rounding.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g12.log
python tools/dfr_variants.py c2 > gpurun_out/var_c2.json 2>gpurun_out/var.err
python tools/dfr_variants.py c4 > gpurun_out/var_c4.json 2>>gpurun_out/var.err
DM_DFR_PIPE=0 python tools/dfr_variants.py c4 > gpurun_out/var_c4_nopipe.json 2>>gpurun_out/var.err

cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_deferred.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g14.log
python tools/dfr_variants.py c2 > gpurun_out/var_c2.json 2>gpurun_out/var.err
python tools/dfr_variants.py c4 > gpurun_out/var_c4.json 2>>gpurun_out/var.err
python tools/dfr_variants.py c2 0 > gpurun_out/var_c2u.json 2>>gpurun_out/var.err

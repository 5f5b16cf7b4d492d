cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g4.log
python tools/dfr_variants.py c2 > gpurun_out/var_c2.json 2>gpurun_out/var.err
python tools/dfr_variants.py c4 > gpurun_out/var_c4.json 2>>gpurun_out/var.err
timeout 900 python tools/dstar.py c2 c3 c4 > gpurun_out/dstar.json 2> gpurun_out/dstar.err

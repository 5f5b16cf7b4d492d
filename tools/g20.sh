cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred.py tests/test_gpu_parity.py tests/test_large_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g20.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g20.log
for c in c4 c2; do timeout 300 python tools/dfr_variants.py $c > gpurun_out/dv_$c.log 2>&1; done

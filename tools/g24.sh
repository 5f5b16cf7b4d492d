cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py tests/test_deferred.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g24.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g24.log
for c in c4 c2; do timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/tl_$c.log 2>&1; done
timeout 600 python tools/c4_step.py c4 deferred 30 > gpurun_out/tl_c4d.log 2>&1

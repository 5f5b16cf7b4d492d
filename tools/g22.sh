cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py tests/test_batch.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g22.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g22.log
for p in 0 1; do for c in c4 c2; do DM_TWO_LOOP_PERSIST=$p timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/tl_${c}_$p.log 2>&1; done; done

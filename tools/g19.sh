cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_batch.py -m gpu -q -x -p no:cacheprovider -k batched > gpurun_out/pytest_g19.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g19.log

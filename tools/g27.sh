cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py tests/test_batch.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g27.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g27.log
for v in 1 0; do
  for c in c4 c2; do DM_STEP_PDL=$v timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/pdl_${v}_$c.log 2>&1; done
done

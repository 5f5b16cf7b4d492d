cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g28.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g28.log
for c in c4 c2; do timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/qm_$c.log 2>&1; done

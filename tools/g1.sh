cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_deferred.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_dfr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dfr.log
for c in c3 c4 c2; do timeout 600 python tools/dfr_probe.py $c 0.3 0.4 0.5 > gpurun_out/probe_$c.json 2> gpurun_out/probe_$c.err; echo "rc=$?" >> gpurun_out/probe_$c.err; done

cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_deferred.py tests/test_large_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g2.log
for c in c2 c4; do timeout 600 python tools/dfr_probe.py $c 0.4 0.5 > gpurun_out/probe_$c.json 2> gpurun_out/probe_$c.err; echo "rc=$?" >> gpurun_out/probe_$c.err; done
timeout 300 python tools/dfr_round.py c2 > gpurun_out/round.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dfr_ -s 1 -c 5 -o gpurun_out/dfr_c2 python tools/dfr_round.py c2 > gpurun_out/ncu_dfr.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_dfr.log

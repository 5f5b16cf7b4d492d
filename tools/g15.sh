cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 300 python tools/dfr_round.py c4 > gpurun_out/round_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dfr_ -s 1 -c 5 -o gpurun_out/r02_dfr_c4_np python tools/dfr_round.py c4 > gpurun_out/ncu_dfr_c4np.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_dfr_c4np.log
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err

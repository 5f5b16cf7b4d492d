cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rounding.py tests/test_batch.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g7.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --schedule deferred > gpurun_out/bench_c5d.json 2> gpurun_out/bench_c5d.err; echo "rc=$?" >> gpurun_out/bench_c5d.err

cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_partition.py tests/test_batch.py tests/test_deferred.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g6.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 600 python bench.py --config c4 --split --steps 20 --warmup 5 > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err; echo "rc=$?" >> gpurun_out/bench_split.err
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err

cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python tools/dstar.py c2 --chunk 0 --iters-exact 300 --iters-deferred 600 > gpurun_out/dstar_c2u.json 2> gpurun_out/dstar_c2u.err
cp profiles/dstar.json gpurun_out/dstar_all.json
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err

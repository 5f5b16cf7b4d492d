# usage (on the GPU box via gpurun): bash tools/run_gpu.sh <steps...>
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for step in "$@"; do
  case "$step" in
    tests) timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
    sweep) timeout 900 python tools/mma_sweep.py c2 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?" >> gpurun_out/sweep.err ;;
    pingpong) ./tools/pingpong > gpurun_out/pingpong.txt 2>&1 ;;
    latency) ./tools/latency > gpurun_out/latency.txt 2>&1 ;;
    trace) timeout 600 python tools/mma_trace.py c2 > gpurun_out/trace.jsonl 2> gpurun_out/trace.err; echo "trace rc=$?" >> gpurun_out/trace.err ;;
    bench) timeout 900 python bench.py --steps 5 --warmup 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err ;;
  esac
done

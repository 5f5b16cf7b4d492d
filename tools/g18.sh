cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-extras --no-ttg --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
for k in mma_np_forward mma_np_backward; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r02_$k $B >> gpurun_out/ncu_mma.log 2>&1; echo "ncu $k rc=$?" >> gpurun_out/ncu_mma.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py -m gpu -q -x -p no:cacheprovider -k "exact_passes or mma_only" > gpurun_out/pytest_g18.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g18.log

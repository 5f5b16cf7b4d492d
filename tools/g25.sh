cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/run_gpu.sh bench_ref
B="python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg --no-extras"
timeout 600 $B > gpurun_out/c4_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_c4_launches.csv $B > gpurun_out/c4_ncu.log 2>&1
for k in mma_np_forward mma_np_backward; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r02_c4full_$k $B >> gpurun_out/c4_ncu.log 2>&1; echo "full $k rc=$?" >> gpurun_out/c4_ncu.log
done

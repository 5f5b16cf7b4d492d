cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/g20.sh
for c in c2 c4; do
  for far in 0 256 1024; do
    DM_MMA_FAR_NS=$far timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-extras --no-ttg --no-e2e --no-cpu-baseline > gpurun_out/far_${c}_$far.json 2> gpurun_out/far_${c}_$far.err
  done
done

# The round's ncu evidence (GPU tool; summarise with tools/ncu_summary.py / ncu_multi.py into
# profiles/r02_final_*): C2 launch lists of the exact and deferred bench step, --set full of the
# exact passes and the argmin walk, the deferred kernels of one round at C2 and C4.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-ttg --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_exact.csv $B > gpurun_out/ncu_le.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_deferred.csv $B --schedule deferred > gpurun_out/ncu_ld.log 2>&1
for k in mma_np_forward mma_np_backward "sweep_backward_kernel<8, 1, 0>" "chunk_step_kernel<1>" k_argmin_walk; do
  n=$(echo "$k" | tr -dc 'a-z_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$(echo $k | sed 's/[<>, ]/./g')" -s 1 -c 1 -o gpurun_out/r02f_$n $B >> gpurun_out/ncu_full.log 2>&1; echo "$k rc=$?" >> gpurun_out/ncu_full.log
done
for c in c2 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dfr_ -s 1 -c 5 -o gpurun_out/r02f_dfr_$c python tools/dfr_round.py $c > gpurun_out/ncu_dfr_$c.log 2>&1
done

cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-ttg --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_exact.csv $B > gpurun_out/ncu_le.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_le.log
timeout 600 $B --schedule deferred > gpurun_out/plain_d.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_deferred.csv $B --schedule deferred > gpurun_out/ncu_ld.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_ld.log
for c in c2 c4; do
timeout 300 python tools/dfr_round.py $c > gpurun_out/round_$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dfr_ -s 1 -c 5 -o gpurun_out/r02_dfr_$c python tools/dfr_round.py $c > gpurun_out/ncu_dfr_$c.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_dfr_$c.log
done
timeout 1200 python -m pytest tests/test_rounding.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g8.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err

# usage (on the GPU box via gpurun): bash tools/run_gpu.sh <step...>
# every output lands in gpurun_out/ (merged back by gpurun)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-ttg --no-e2e --no-cpu-baseline"
for step in "$@"; do
  case "$step" in
    tests) timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
    bench) timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/bench_default.err ;;
    bench_ref) timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err ;;
    bench_c5) timeout 900 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err ;;
    bench_split) timeout 600 python bench.py --config c4 --split --steps 20 --warmup 5 > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err ;;
    dstar) timeout 1500 python tools/dstar.py c2 c3 c4 > gpurun_out/dstar.json 2> gpurun_out/dstar.err
           timeout 1200 python tools/dstar.py c2 --chunk 0 --iters-exact 300 --iters-deferred 600 >> gpurun_out/dstar.json 2>> gpurun_out/dstar.err
           cp profiles/dstar.json gpurun_out/dstar_all.json ;;
    ncu_list)  # launch lists of the exact and the deferred bench step (profiles/r02_launches_*.md)
      timeout 600 $B > gpurun_out/plain.log 2>&1 && \
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_exact.csv $B > gpurun_out/ncu_le.log 2>&1
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_deferred.csv $B --schedule deferred > gpurun_out/ncu_ld.log 2>&1 ;;
    ncu_dfr)  # one deferred round at C2 and C4 (profiles/r02_dfr_*_full.md via tools/ncu_multi.py)
      for c in c2 c4; do
        timeout 300 python tools/dfr_round.py $c > gpurun_out/round_$c.log 2>&1 && \
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:dfr_ -s 1 -c 5 -o gpurun_out/r02_dfr_$c python tools/dfr_round.py $c > gpurun_out/ncu_dfr_$c.log 2>&1
      done ;;
    ncu_mma)  # the exact passes at C2
      timeout 600 $B > gpurun_out/plain.log 2>&1 && \
      for k in mma_np_forward mma_np_backward; do
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r02_$k $B >> gpurun_out/ncu_mma.log 2>&1
      done ;;
    variants) for c in c2 c4; do python tools/dfr_variants.py $c > gpurun_out/var_$c.json 2>>gpurun_out/var.err; done ;;
    hints) for c in c2 c4; do python tools/ab_hints.py $c > gpurun_out/ab_hints_$c.json 2>>gpurun_out/ab_hints.err; done ;;
    c5_phases) timeout 900 python tools/c5_phases.py > gpurun_out/c5_phases.jsonl 2> gpurun_out/c5_phases.err ;;
    probe) for c in c3 c4 c2; do timeout 600 python tools/dfr_probe.py $c 0.4 0.5 > gpurun_out/probe_$c.json 2> gpurun_out/probe_$c.err; done ;;
    profile) bash tools/profile_round.sh ;;  # the final-round ncu captures (profiles/r02_final_*)
    c5_batched) timeout 900 python tools/c5_batched.py 64 exact > gpurun_out/c5_batched.log 2>&1 ;;
    steps) for c in c4 c2; do timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/step_$c.log 2>&1; done ;;
    *) echo "unknown step $step" ;;
  esac
done

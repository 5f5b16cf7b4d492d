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
    ncu_list)
      B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg"
      timeout 900 $B > gpurun_out/plain.log 2>&1 && \
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
          --log-file gpurun_out/launches.csv $B > gpurun_out/ncu.log 2>&1; echo "ncu_list rc=$?" >> gpurun_out/ncu.log ;;
    ncu_full)
      B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg"
      timeout 900 $B > gpurun_out/plain.log 2>&1 && \
      for k in mma_np_forward mma_np_backward sweep_backward chunk_step_kernel k_argmin; do
        timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
            -o gpurun_out/full_$k $B >> gpurun_out/ncu_full.log 2>&1; echo "ncu_full $k rc=$?" >> gpurun_out/ncu_full.log
      done ;;
    ncu_mma2)
      B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg"
      timeout 900 $B > gpurun_out/plain.log 2>&1 && \
      for k in mma_np_forward mma_np_backward; do
        timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
            -o gpurun_out/full_$k $B >> gpurun_out/ncu_full.log 2>&1; echo "ncu_full $k rc=$?" >> gpurun_out/ncu_full.log
      done ;;
    ncu_mma)
      B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ttg"
      timeout 900 $B > gpurun_out/plain.log 2>&1 && \
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mma_forward -s 1 -c 1 \
          -o gpurun_out/prof_mma_fw $B > gpurun_out/ncu_mma.log 2>&1 && \
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mma_backward -s 1 -c 1 \
          -o gpurun_out/prof_mma_bw $B >> gpurun_out/ncu_mma.log 2>&1; echo "ncu_mma rc=$?" >> gpurun_out/ncu_mma.log ;;
    ab) timeout 1200 python tools/ab_mma.py tools/ab/*.so tools/ab/*.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err ;;
    abdesc) timeout 1200 python tools/ab_mma.py DM_MMA_DESC=0 DM_MMA_DESC=1 DM_MMA_DESC=0 DM_MMA_DESC=1 > gpurun_out/abdesc.jsonl 2> gpurun_out/abdesc.err ;;
    abnp) timeout 1200 python tools/ab_mma.py DM_MMA_NP=0 DM_MMA_NP=1 DM_MMA_NP=0 DM_MMA_NP=1 > gpurun_out/abnp.jsonl 2> gpurun_out/abnp.err ;;
    e2eprof) timeout 900 python tools/e2e_profile.py > gpurun_out/e2eprof.txt 2>&1 ;;
    create) timeout 900 python tools/create_timing.py > gpurun_out/create.txt 2>&1 ;;
    workbench) ./tools/workbench > gpurun_out/workbench.jsonl 2>&1 ;;
    worklat) timeout 600 python tools/work_latency.py icosa > gpurun_out/worklat.txt 2>&1 ;;
    timeline) timeout 900 python tools/timeline.py > gpurun_out/timeline.json 2> gpurun_out/timeline.err ;;
    concur) timeout 900 python tools/concurrency.py > gpurun_out/concur.jsonl 2> gpurun_out/concur.err ;;
    batch) timeout 1500 python tools/batch_solve.py 4 > gpurun_out/batch.jsonl 2> gpurun_out/batch.err ;;
    phases) timeout 900 python tools/step_phases.py 12 > gpurun_out/phases.jsonl 2> gpurun_out/phases.err ;;
    vec) timeout 300 python tools/vec_bench.py > gpurun_out/vec.json 2> gpurun_out/vec.err && \
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv \
          --log-file gpurun_out/vec_launches.csv python tools/vec_bench.py > gpurun_out/vec_ncu.log 2>&1 ;;
    prof) timeout 900 python tools/step_profile.py > gpurun_out/step_profile.txt 2>&1 ;;
    sampler) timeout 900 python tools/sampler_cost.py > gpurun_out/sampler.txt 2>&1 ;;
  esac
done

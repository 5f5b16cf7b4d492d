cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g26.log
for v in ring noring; do
  L=""; [ $v = noring ] && L="DM_LIB_PATH=paper_2310_08230_b200/_ab/noring.so"
  for c in c4 c2; do env $L timeout 600 python tools/c4_step.py $c exact 20 > gpurun_out/rs_${v}_$c.log 2>&1; done
  env $L timeout 300 python tools/dfr_variants.py c4 > gpurun_out/rs_${v}_dv.log 2>&1
done

mkdir -p gpurun_out/datasets
timeout 900 python -m pytest tests/test_live_gpu.py -q --timeout 400 -k "coulomb or nbody" > gpurun_out/rsq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rsq_pytest.log
tail -n 2 gpurun_out/rsq_pytest.log
if grep -q "rc=0" gpurun_out/rsq_pytest.log; then
  timeout 1500 python scripts/live_sweep.py --bench nbody --update datasets/nbody-b200 --select FAST_RSQRT=1 \
      --out gpurun_out/datasets/nbody-b200 > gpurun_out/datasets/nbody_upd.log 2>&1
  tail -n 1 gpurun_out/datasets/nbody_upd.log | cut -c1-900
  timeout 600 python scripts/live_sweep.py --bench coulomb --update datasets/coulomb-b200 --select USE_CONST=0 \
      --out gpurun_out/datasets/coulomb-b200 > gpurun_out/datasets/coulomb_upd.log 2>&1
  tail -n 1 gpurun_out/datasets/coulomb_upd.log | cut -c1-900
  for b in nbody coulomb; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${b}\$" -s 1 -c 1 \
        -o gpurun_out/kb_${b}2 python scripts/run_variant.py --bench $b --best gpurun_out/datasets/${b}-b200 > gpurun_out/kb_${b}2.log 2>&1
    tail -n 1 gpurun_out/kb_${b}2.log
  done
fi

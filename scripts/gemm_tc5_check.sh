# validate + time the tcgen05 GEMM variants; re-measure them into the dataset
mkdir -p gpurun_out/datasets
timeout 900 python -m pytest tests/test_live_gpu.py -q --timeout 400 -k "gemm" > gpurun_out/tc5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tc5_pytest.log
tail -n 2 gpurun_out/tc5_pytest.log
if grep -q "rc=0" gpurun_out/tc5_pytest.log; then
  python scripts/run_variant.py --bench gemm --index 5664 --launches 5
  timeout 900 python scripts/live_sweep.py --bench gemm --update datasets/gemm-b200 --select tc5 \
      --out gpurun_out/datasets/gemm-b200 > gpurun_out/datasets/gemm_tc5.log 2>&1
  tail -n 1 gpurun_out/datasets/gemm_tc5.log | cut -c1-900
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^gemm\$" -s 1 -c 1 \
      -o gpurun_out/kb_gemm3 python scripts/run_variant.py --bench gemm --best gpurun_out/datasets/gemm-b200 > gpurun_out/kb_gemm3.log 2>&1
  tail -n 1 gpurun_out/kb_gemm3.log
fi

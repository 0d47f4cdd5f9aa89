# validate the conv / nbody kernel changes, draw sub-phase clocks, nbody sweep, conv re-measure
mkdir -p gpurun_out/datasets
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r5_pytest.log
tail -n 3 gpurun_out/r5_pytest.log
CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python bench.py --steps 1 --warmup 3 --kernel-only 2>&1 | grep -E "clk" | head -6 > gpurun_out/r5_clk.log; cat gpurun_out/r5_clk.log
if grep -q "rc=0" gpurun_out/r5_pytest.log; then
  timeout 1700 python scripts/live_sweep.py --bench nbody --out gpurun_out/datasets/nbody-b200 \
      --checkpoint gpurun_out/datasets/nbody3.ckpt.npz --budget-s 1300 > gpurun_out/datasets/nbody.log 2>&1
  echo "nbody rc=$?"; tail -n 1 gpurun_out/datasets/nbody.log | cut -c1-800
  timeout 1000 python scripts/live_sweep.py --bench conv --update datasets/conv-b200 --select LOCAL=1 \
      --out gpurun_out/datasets/conv-b200 > gpurun_out/datasets/conv_l1.log 2>&1
  tail -n 1 gpurun_out/datasets/conv_l1.log | cut -c1-800
  timeout 1000 python scripts/live_sweep.py --bench conv --update gpurun_out/datasets/conv-b200 --select LOCAL=2 \
      --out gpurun_out/datasets/conv-b200 > gpurun_out/datasets/conv_l2.log 2>&1
  tail -n 1 gpurun_out/datasets/conv_l2.log | cut -c1-800
fi

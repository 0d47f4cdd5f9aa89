# validate the conv kernel, re-measure the variants whose code changed, ncu the new best
mkdir -p gpurun_out/datasets
timeout 900 python -m pytest tests/test_live_gpu.py -q --timeout 400 -k "conv" > gpurun_out/conv_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/conv_pytest.log
tail -n 2 gpurun_out/conv_pytest.log
if grep -q "rc=0" gpurun_out/conv_pytest.log; then
  timeout 1500 python scripts/live_sweep.py --bench conv --update datasets/conv-b200 --select ${1:-CACHE_F=0} \
      --out gpurun_out/datasets/conv-b200 > gpurun_out/datasets/conv_upd.log 2>&1
  tail -n 1 gpurun_out/datasets/conv_upd.log | cut -c1-900
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^conv\$" -s 1 -c 1 \
      -o gpurun_out/kb_conv2 python scripts/run_variant.py --bench conv --best gpurun_out/datasets/conv-b200 > gpurun_out/kb_conv2.log 2>&1
  tail -n 1 gpurun_out/kb_conv2.log
fi

mkdir -p gpurun_out/datasets
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r6_pytest.log
tail -n 3 gpurun_out/r6_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --kernel-only 2>&1 | grep "\[bench\]"
CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python bench.py --steps 1 --warmup 3 --kernel-only 2>&1 | grep -E "clk" | head -4
cp -f datasets/ckpt/nbody.ckpt.npz gpurun_out/datasets/nbody3.ckpt.npz
timeout 900 python scripts/live_sweep.py --bench nbody --out gpurun_out/datasets/nbody-b200 \
    --checkpoint gpurun_out/datasets/nbody3.ckpt.npz --budget-s 600 > gpurun_out/datasets/nbody.log 2>&1
tail -n 1 gpurun_out/datasets/nbody.log | cut -c1-600
timeout 1500 python scripts/live_experiment.py datasets/transpose-b200 datasets/coulomb-b200 datasets/conv-b200 datasets/gemm-b200 gpurun_out/datasets/nbody-b200 --out gpurun_out/r6_experiments_replay.json > gpurun_out/r6_experiments.log 2>&1
tail -n 5 gpurun_out/r6_experiments.log | cut -c1-900

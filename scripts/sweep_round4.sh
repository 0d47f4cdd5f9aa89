# finish nbody, re-measure the tcgen05 gemm variants, replay experiments on all five spaces
mkdir -p gpurun_out/datasets
cp -f datasets/ckpt/nbody.ckpt.npz gpurun_out/datasets/nbody2.ckpt.npz
timeout 1500 python scripts/live_sweep.py --bench nbody --out gpurun_out/datasets/nbody-b200 \
    --checkpoint gpurun_out/datasets/nbody2.ckpt.npz --budget-s 1100 > gpurun_out/datasets/nbody.log 2>&1
echo "nbody rc=$?"; tail -n 1 gpurun_out/datasets/nbody.log | cut -c1-800
timeout 900 python scripts/live_sweep.py --bench gemm --update datasets/gemm-b200 --select tc5 \
    --out gpurun_out/datasets/gemm-b200 > gpurun_out/datasets/gemm_tc5.log 2>&1
echo "tc5 rc=$?"; tail -n 1 gpurun_out/datasets/gemm_tc5.log | cut -c1-900

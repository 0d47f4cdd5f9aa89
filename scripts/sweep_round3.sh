# nbody (new j-split kernel) full sweep, gemm resume + re-measure of the tcgen05 variants
mkdir -p gpurun_out/datasets
timeout 2000 python scripts/live_sweep.py --bench nbody --out gpurun_out/datasets/nbody-b200 \
    --checkpoint gpurun_out/datasets/nbody2.ckpt.npz --budget-s 1300 > gpurun_out/datasets/nbody.log 2>&1
echo "nbody rc=$?"; tail -n 1 gpurun_out/datasets/nbody.log | cut -c1-700
cp -f datasets/ckpt/gemm.ckpt.npz gpurun_out/datasets/gemm.ckpt.npz
timeout 1200 python scripts/live_sweep.py --bench gemm --out gpurun_out/datasets/gemm-b200 \
    --checkpoint gpurun_out/datasets/gemm.ckpt.npz --budget-s 800 > gpurun_out/datasets/gemm.log 2>&1
echo "gemm rc=$?"; tail -n 1 gpurun_out/datasets/gemm.log | cut -c1-700
timeout 900 python scripts/live_sweep.py --bench gemm --update gpurun_out/datasets/gemm-b200 --select tc5 \
    --out gpurun_out/datasets/gemm-b200 > gpurun_out/datasets/gemm_tc5.log 2>&1
echo "tc5 rc=$?"; tail -n 1 gpurun_out/datasets/gemm_tc5.log | cut -c1-900

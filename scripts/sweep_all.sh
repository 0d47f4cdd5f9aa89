# exhaustive B200 sweeps of the five benchmark spaces at the paper's sizes
# usage: bash scripts/sweep_all.sh [bench ...]
mkdir -p gpurun_out/datasets
for b in ${@:-coulomb transpose nbody conv gemm}; do
  timeout 1500 python scripts/live_sweep.py --bench $b --out gpurun_out/datasets/$b-b200 \
      --checkpoint gpurun_out/datasets/$b.ckpt.npz > gpurun_out/datasets/$b.log 2>&1
  echo "$b rc=$?" >> gpurun_out/datasets/$b.log
  tail -n 2 gpurun_out/datasets/$b.log
done

# One clean exhaustive re-sweep of every B200 dataset with the round's final
# kernels: the five paper-size spaces and the
# five second input sizes of the input-portability study (PAPER.md:678-695,
# 745).  Timed (median of 3, L2 flushed) and profiled (24 Table-1 metrics).
# usage: bash scripts/resweep_r02.sh [name ...]   (checkpointed; re-run resumes)
mkdir -p gpurun_out/datasets
run() {  # name bench size
  timeout 3000 python scripts/live_sweep.py --bench $2 ${3:+--size $3} --out gpurun_out/datasets/$1-b200 \
      --checkpoint gpurun_out/datasets/$1.ckpt.npz > gpurun_out/datasets/$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/datasets/$1.log
  tail -n 2 gpurun_out/datasets/$1.log | cut -c1-300
}
for x in ${@:-coulomb transpose nbody gemm conv nbody-131072 gemm-128 gemm-16x4096 gemm-4096x16 conv-8192}; do
  case $x in
    coulomb|transpose|nbody|gemm|conv) run $x $x "" ;;
    gemm-128) run $x gemm m=128,n=128,k=128 ;;
    gemm-16x4096) run $x gemm m=16,n=4096,k=4096 ;;
    gemm-4096x16) run $x gemm m=4096,n=16,k=4096 ;;
    conv-8192) run $x conv width=8192,height=8192 ;;
    nbody-131072) run $x nbody bodies=131072 ;;
    nbody-32768) run $x nbody bodies=32768 ;;
  esac
done

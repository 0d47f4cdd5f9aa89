# exhaustive B200 sweeps at the second input sizes of the input-portability
# study (BASELINE config 4): n-body 131,072 bodies,
# conv 8192^2, GEMM 128^2 / 16x4096 / 4096x16 (configurations that do not
# tile the input are not in its space)
# usage: bash scripts/sweep_cross.sh [name ...]
mkdir -p gpurun_out/datasets
run() {  # name bench size
  timeout 2400 python scripts/live_sweep.py --bench $2 --size $3 --out gpurun_out/datasets/$1-b200 \
      --checkpoint gpurun_out/datasets/$1.ckpt.npz > gpurun_out/datasets/$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/datasets/$1.log
  tail -n 2 gpurun_out/datasets/$1.log | cut -c1-400
}
for x in ${@:-gemm-128 gemm-16x4096 gemm-4096x16 conv-8192 nbody-131072}; do
  case $x in
    gemm-128) run $x gemm m=128,n=128,k=128 ;;
    gemm-16x4096) run $x gemm m=16,n=4096,k=4096 ;;
    gemm-4096x16) run $x gemm m=4096,n=16,k=4096 ;;
    conv-8192) run $x conv width=8192,height=8192 ;;
    nbody-131072) run $x nbody bodies=131072 ;;
  esac
done

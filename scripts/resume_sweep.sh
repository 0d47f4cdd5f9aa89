# Resume a checkpointed sweep across gpurun calls: gpurun_out/ does not travel
# to the box, datasets/ckpt/ (git-ignored) does.
#   bash scripts/resume_sweep.sh <name> <bench> [size] [budget_s]
name=$1; bench=$2; size=$3; budget=${4:-3000}
mkdir -p gpurun_out/datasets
[ -f datasets/ckpt/$name.ckpt.npz ] && cp datasets/ckpt/$name.ckpt.npz gpurun_out/datasets/$name.ckpt.npz
timeout $((budget + 600)) python scripts/live_sweep.py --bench $bench ${size:+--size $size} \
    --out gpurun_out/datasets/$name-b200 --checkpoint gpurun_out/datasets/$name.ckpt.npz \
    --budget-s $budget > gpurun_out/datasets/$name.log 2>&1
echo "$name rc=$?" >> gpurun_out/datasets/$name.log
tail -n 3 gpurun_out/datasets/$name.log | cut -c1-300

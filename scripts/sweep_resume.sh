# resume exhaustive sweeps from checkpoints under datasets/ckpt (pushed with
# the repo); each benchmark gets a measuring budget so its dataset is always
# written before the call's limit
# usage: bash scripts/sweep_resume.sh "<bench>:<budget_s> ..."
mkdir -p gpurun_out/datasets
for spec in $1; do
  b=${spec%%:*}; budget=${spec##*:}
  cp -f datasets/ckpt/$b.ckpt.npz gpurun_out/datasets/$b.ckpt.npz 2>/dev/null
  timeout $((budget + 600)) python scripts/live_sweep.py --bench $b --out gpurun_out/datasets/$b-b200 \
      --checkpoint gpurun_out/datasets/$b.ckpt.npz --budget-s $budget > gpurun_out/datasets/$b.log 2>&1
  echo "$b rc=$?" >> gpurun_out/datasets/$b.log
  tail -n 2 gpurun_out/datasets/$b.log | cut -c1-400
done

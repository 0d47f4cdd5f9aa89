# round-2 final evidence B: profiled-step cost on every space, live searches
# (10 per searcher, full 24-metric profile and the labelled single-pass mode)
# and ncu captures of the sweeps' best benchmark kernels
TAG=${1:-r02t}
mkdir -p gpurun_out
timeout 1200 python scripts/profile_cost.py --reps 3 > gpurun_out/${TAG}_profile_cost.jsonl 2> gpurun_out/${TAG}_profile_cost.err
timeout 2400 python scripts/live_experiment.py datasets/coulomb-b200 datasets/nbody-b200 datasets/transpose-b200 --live 10 --out gpurun_out/${TAG}_live_full.json > gpurun_out/${TAG}_live_full.log 2>&1
timeout 2400 python scripts/live_experiment.py datasets/coulomb-b200 datasets/nbody-b200 datasets/transpose-b200 --live 10 --mode group1 --out gpurun_out/${TAG}_live_group1.json > gpurun_out/${TAG}_live_group1.log 2>&1
bash scripts/ncu_benchmarks.sh > gpurun_out/${TAG}_kb.log 2>&1
for b in transpose coulomb nbody conv gemm; do
  python scripts/ncu_summary.py --full gpurun_out/kb_${b}.ncu-rep --title "${TAG}: ${b}, best configuration of the round-2 sweep" --out gpurun_out/${TAG}_kb_${b}.md > /dev/null 2>&1
done
rm -f gpurun_out/kb_*.ncu-rep
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl; do echo "== $f"; tail -n 8 "$f" | cut -c1-400; done

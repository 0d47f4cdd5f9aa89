TAG=${1:-r02v}
mkdir -p gpurun_out
timeout 900 python scripts/live_experiment.py datasets/coulomb-b200 datasets/transpose-b200 datasets/nbody-b200 datasets/conv-b200 datasets/gemm-b200 --measured-overhead --out gpurun_out/${TAG}_replay.json > gpurun_out/${TAG}_replay.log 2>&1
timeout 1800 bash scripts/sanitize.sh ${TAG} > gpurun_out/${TAG}_sanitize.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
rm -rf gpurun_out/sanitizer_${TAG}/*_racecheck.log.big 2>/dev/null; du -sh gpurun_out
for f in gpurun_out/${TAG}_*.log gpurun_out/sanitizer_${TAG}/summary.txt; do echo "== $f"; tail -n 12 "$f" | cut -c1-300; done

# final check of the round's tree: all GPU tests, smoke, bench, and the
# sanitizer over the re-decision and the tiled path
TAG=${1:-r02ac}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
mkdir -p gpurun_out/sanitizer_${TAG}
for c in seq tiled hg; do for tool in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py $c > gpurun_out/sanitizer_${TAG}/${c}_${tool}.log 2>&1
  echo "$c $tool rc=$?" >> gpurun_out/sanitizer_${TAG}/summary.txt
done; done
for f in gpurun_out/${TAG}_*.log gpurun_out/sanitizer_${TAG}/summary.txt; do echo "== $f"; tail -n 5 "$f" | cut -c1-300; done

# compute-sanitizer over every device path (scripts/sanitize_cases.py)
# usage: bash scripts/sanitize.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/sanitizer_${TAG}
mkdir -p $OUT
for c in scratch ws hg topk report tiled seq mq; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py $c > $OUT/${c}_${tool}.log 2>&1
    echo "$c $tool rc=$?" | tee -a $OUT/summary.txt
  done
done
# the live path: CUPTI replay does not run under the sanitizer's own
# instrumentation, so libct_tune gets memcheck only
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py tune > $OUT/tune_memcheck.log 2>&1
echo "tune memcheck rc=$?" | tee -a $OUT/summary.txt

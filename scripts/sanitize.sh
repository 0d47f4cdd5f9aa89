# compute-sanitizer over every device path (scripts/sanitize_cases.py)
# usage: bash scripts/sanitize.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/sanitizer_${TAG}
mkdir -p $OUT
for c in scratch ws hg topk report tiled seq; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py $c > $OUT/${c}_${tool}.log 2>&1
    echo "$c $tool rc=$?" | tee -a $OUT/summary.txt
  done
done
# the live path: CUPTI cannot subscribe next to the sanitizer
# (CUPTI_ERROR_MULTIPLE_SUBSCRIBERS_NOT_SUPPORTED), so libct_tune's compile,
# launch and timing path gets memcheck, the collector none
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py tune > $OUT/tune_memcheck.log 2>&1
echo "tune memcheck rc=$?" | tee -a $OUT/summary.txt

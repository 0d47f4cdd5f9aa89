# After a B200 re-sweep (scripts/resweep_r02.sh): install the datasets from
# gpurun_out/datasets/ and re-record every reference golden that reads them,
# with the REFERENCE implementation (build container only: imports
# /root/reference).
#   bash scripts/regen_b200_goldens.sh
set -e
for d in gpurun_out/datasets/*-b200; do
  name=$(basename $d)
  [ -f $d/measurements.csv ] || continue
  mkdir -p datasets/$name
  cp $d/space.csv $d/measurements.csv $d/arch.txt $d/sweep_summary.json datasets/$name/
  echo "installed $name"
done
export PYTHONPATH=/root/reference/pkg/src
python tests/golden/make_b200_golden.py
python tests/golden/make_b200_models_golden.py
python tests/golden/make_topk_golden.py
python tests/golden/make_order_golden.py
python tests/golden/make_cross_golden.py

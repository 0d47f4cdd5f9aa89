TAG=${1:-r02u}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cupti_gpu.py tests/test_live_gpu.py -q --timeout 600 -rs > gpurun_out/${TAG}_pytest_live.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_live.log
timeout 2400 python -X faulthandler scripts/live_experiment.py datasets/coulomb-b200 datasets/nbody-b200 datasets/transpose-b200 --live 10 --out gpurun_out/${TAG}_live_full.json > gpurun_out/${TAG}_live_full.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_full.log
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 8 "$f" | cut -c1-300; done

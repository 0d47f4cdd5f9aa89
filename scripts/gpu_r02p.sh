TAG=${1:-r02p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cupti_gpu.py tests/test_live_gpu.py -q --timeout 600 -rs > gpurun_out/${TAG}_pytest_live.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_live.log
# batched-profile sweep speed on a small space (timing + 24 metrics)
timeout 900 python scripts/live_sweep.py --bench coulomb --out gpurun_out/${TAG}_coulomb_sweep > gpurun_out/${TAG}_coulomb_sweep.log 2>&1
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 15 "$f" | cut -c1-400; done

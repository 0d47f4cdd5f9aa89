TAG=${1:-r02i}
mkdir -p gpurun_out/tsweep_i
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_live_gpu.py -q --timeout 600 -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1500 python scripts/search_sweep.py --nt auto --spaces gemm_full,stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_tiled_sweep.jsonl 2> gpurun_out/${TAG}_tiled_sweep.err; echo "rc=$?" >> gpurun_out/${TAG}_tiled_sweep.err
for b in nbody conv; do
  timeout 1800 python scripts/live_sweep.py --bench $b --out gpurun_out/tsweep_i/$b --no-profile > gpurun_out/tsweep_i/$b.log 2>&1; echo "rc=$?" >> gpurun_out/tsweep_i/$b.log
done
timeout 600 python -X faulthandler scripts/profile_cost.py --reps 3 > gpurun_out/${TAG}_profile_cost.jsonl 2> gpurun_out/${TAG}_profile_cost.err; echo "rc=$?" >> gpurun_out/${TAG}_profile_cost.err
for f in gpurun_out/${TAG}_* gpurun_out/tsweep_i/*.log; do echo "== $f"; tail -n 12 "$f" | cut -c1-500; done

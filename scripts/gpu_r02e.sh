# round-2 evidence: GPU tests, profiled-step cost, time-only sweeps of the
# compute-bound spaces (new best configurations after the FFMA2/TMA kernel
# changes), stress-size search sweep + one full ncu capture at 1M configs
TAG=${1:-r02e}
mkdir -p gpurun_out/tsweep
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python scripts/profile_cost.py > gpurun_out/${TAG}_profile_cost.jsonl 2> gpurun_out/${TAG}_profile_cost.err; echo "rc=$?" >> gpurun_out/${TAG}_profile_cost.err
timeout 1200 python scripts/search_sweep.py --nt auto --spaces stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 3 > gpurun_out/${TAG}_stress_sweep.jsonl 2> gpurun_out/${TAG}_stress_sweep.err; echo "rc=$?" >> gpurun_out/${TAG}_stress_sweep.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_stress_full python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 10 --kernel-only > gpurun_out/${TAG}_ncu_stress.log 2>&1
for b in nbody conv gemm coulomb; do
  timeout 1800 python scripts/live_sweep.py --bench $b --out gpurun_out/tsweep/$b --no-profile > gpurun_out/tsweep/$b.log 2>&1; echo "rc=$?" >> gpurun_out/tsweep/$b.log
done
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.err gpurun_out/tsweep/*.log; do echo "== $f"; tail -n 4 "$f" | cut -c1-700; done

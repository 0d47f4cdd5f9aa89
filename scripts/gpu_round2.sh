# round-2 evidence session: GPU tests, smoke, bench, per-space + stress sweep,
# ncu launch list and full captures (bench kernel, stress kernel), phase
# clocks, the FFMA2 micro-benchmark and the profiled-step cost breakdown
# usage: bash scripts/gpu_round2.sh <tag>
TAG=${1:-r02b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
./scripts/micro/ffma2_rate > gpurun_out/${TAG}_ffma2.log 2>&1
timeout 1500 python -m pytest tests/test_live_gpu.py tests/test_cupti_gpu.py -q --timeout 600 -rs > gpurun_out/${TAG}_pytest_live.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_live.log
timeout 900 python scripts/profile_cost.py > gpurun_out/${TAG}_profile_cost.jsonl 2> gpurun_out/${TAG}_profile_cost.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs --deselect tests/test_live_gpu.py --deselect tests/test_cupti_gpu.py > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 1200 python scripts/search_sweep.py --nt auto --spaces b200:coulomb,b200:transpose,b200:nbody,b200:conv,b200:gemm,gemm_full,stress:1048576,stress:4194304 --runs 3 > gpurun_out/${TAG}_search_sweep.jsonl 2> gpurun_out/${TAG}_search_sweep.err; echo "sweep rc=$?" >> gpurun_out/${TAG}_search_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_search_full python bench.py --steps 1 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_stress_full python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 10 --kernel-only > gpurun_out/${TAG}_ncu_stress.log 2>&1
CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python bench.py --steps 1 --warmup 3 --kernel-only > gpurun_out/${TAG}_clk.log 2>&1
for r in 148 444 1000; do CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python scripts/search_sweep.py --nt auto --spaces b200:transpose --reps $r --runs 1 > gpurun_out/${TAG}_clk_r$r.log 2>&1; done
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.err; do echo "== $f"; tail -n 3 "$f" | cut -c1-600; done

# one GPU evidence session: parity tests, smoke, bench, ncu launch list + full capture
# usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r01f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_search_full python bench.py --steps 1 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_full.log 2>&1
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-600; done

# round-2 final evidence A: GPU tests, smoke, bench (both arms), ncu of the
# bench kernel and of the tiled path at 1M, per-space search sweep, the
# cross-input improvement matrix
TAG=${1:-r02s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/${TAG}_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_search_full python bench.py --steps 1 --warmup 3 --kernel-only > gpurun_out/${TAG}_ncu_full.log 2>&1
CT_SEARCH_TILED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled_score -c 1 -o gpurun_out/${TAG}_tiled_score python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 2 --kernel-only > gpurun_out/${TAG}_ncu_ts.log 2>&1
CT_SEARCH_TILED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled_weights -c 1 -o gpurun_out/${TAG}_tiled_weights python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 2 --kernel-only > gpurun_out/${TAG}_ncu_tw.log 2>&1
timeout 1500 python scripts/search_sweep.py --nt auto --spaces b200:coulomb,b200:transpose,b200:nbody,b200:conv,b200:gemm,gemm_full --runs 5 > gpurun_out/${TAG}_search_sweep.jsonl 2> gpurun_out/${TAG}_search_sweep.err
timeout 1500 python scripts/search_sweep.py --nt auto --spaces stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 >> gpurun_out/${TAG}_search_sweep.jsonl 2>> gpurun_out/${TAG}_search_sweep.err
CT_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_2rank_shared.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_2rank_shared.log
timeout 1500 python scripts/cross_matrix.py --out gpurun_out/${TAG}_cross_input.json > gpurun_out/${TAG}_cross.log 2>&1
# ncu reports are summarised on the box (gpurun_out must stay under 64 MiB)
python scripts/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv --full gpurun_out/${TAG}_search_full.ncu-rep --title "${TAG}: k_profile_search, bench workload" --out gpurun_out/${TAG}_search.md > /dev/null 2>&1
python scripts/ncu_summary.py --full gpurun_out/${TAG}_tiled_score.ncu-rep --title "${TAG}: k_tiled_score, stress 1M, R=444" --out gpurun_out/${TAG}_tiled_score.md > /dev/null 2>&1
python scripts/ncu_summary.py --full gpurun_out/${TAG}_tiled_weights.ncu-rep --title "${TAG}: k_tiled_weights, stress 1M, R=444" --out gpurun_out/${TAG}_tiled_weights.md > /dev/null 2>&1
rm -f gpurun_out/${TAG}_tiled_score.ncu-rep gpurun_out/${TAG}_tiled_weights.ncu-rep
du -sh gpurun_out
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl; do echo "== $f"; tail -n 6 "$f" | cut -c1-400; done

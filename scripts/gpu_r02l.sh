TAG=${1:-r02l}
mkdir -p gpurun_out
./scripts/micro/ffma2_rate > gpurun_out/${TAG}_ffma2.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 1500 python scripts/search_sweep.py --nt auto --spaces stress:16384,stress:65536,gemm_full --reps 1000 --outer 40 --runs 3 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_nsweep_small.jsonl 2> gpurun_out/${TAG}_nsweep_small.err
timeout 1500 python scripts/search_sweep.py --nt auto --spaces stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_nsweep_large.jsonl 2> gpurun_out/${TAG}_nsweep_large.err
CT_TUNE_TRACE=1 timeout 300 python scripts/profile_cost.py --benches transpose --reps 2 > gpurun_out/${TAG}_trace_user.jsonl 2> gpurun_out/${TAG}_trace_user.err
CT_TUNE_TRACE=1 python scripts/profile_cost.py --one transpose:all24 --reps 2 > gpurun_out/${TAG}_trace_user_one.log 2>&1
CT_TUNE_REPLAY=kernel timeout 600 python scripts/profile_cost.py --benches transpose,coulomb,gemm --reps 3 > gpurun_out/${TAG}_profile_cost_kernel_replay.jsonl 2> gpurun_out/${TAG}_pck.err
timeout 1500 bash scripts/sanitize.sh ${TAG} > gpurun_out/${TAG}_sanitize.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl gpurun_out/sanitizer_${TAG}/summary.txt; do echo "== $f"; tail -n 25 "$f" | cut -c1-300; done

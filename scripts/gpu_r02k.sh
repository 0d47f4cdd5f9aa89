TAG=${1:-r02k}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -q --timeout 900 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1200 python scripts/search_sweep.py --nt auto --spaces gemm_full,stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_tiled_sweep.jsonl 2> gpurun_out/${TAG}_tiled_sweep.err
CT_SEARCH_TILED=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_tiled_launches.csv python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 3 --runs 1 > gpurun_out/${TAG}_ncu_tl.log 2>&1
timeout 2400 bash scripts/sanitize.sh ${TAG} > gpurun_out/${TAG}_sanitize.log 2>&1
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl gpurun_out/sanitizer_${TAG}/summary.txt; do echo "== $f"; tail -n 40 "$f" | cut -c1-300; done

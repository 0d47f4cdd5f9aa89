TAG=${1:-r02x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "sequential or gemm_full or stress or tiled" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1200 python scripts/search_sweep.py --nt auto --spaces gemm_full,stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 3 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err
CT_SEARCH_TILED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_tiled_launches.csv python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 10 --kernel-only > gpurun_out/${TAG}_ncu.log 2>&1
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl; do echo "== $f"; tail -n 8 "$f" | cut -c1-300; done

TAG=${1:-r02j}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1200 python scripts/search_sweep.py --nt auto --spaces gemm_full,stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_tiled_sweep.jsonl 2> gpurun_out/${TAG}_tiled_sweep.err
CT_SEARCH_TILED=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_tiled_launches.csv python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 2 --kernel-only > gpurun_out/${TAG}_ncu_tl.log 2>&1
CT_SEARCH_TILED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled_score -s 3 -c 1 -o gpurun_out/${TAG}_tiled_score python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 2 --kernel-only > gpurun_out/${TAG}_ncu_ts.log 2>&1
CT_SEARCH_TILED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled_weights -s 3 -c 1 -o gpurun_out/${TAG}_tiled_weights python scripts/search_sweep.py --nt auto --spaces stress:1048576 --reps 444 --outer 2 --kernel-only > gpurun_out/${TAG}_ncu_tw.log 2>&1
for b in "nbody 1776" "conv 2282"; do set -- $b
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$1\$" -s 1 -c 1 -o gpurun_out/${TAG}_kb_$1 python scripts/run_variant.py --bench $1 --index $2 > gpurun_out/${TAG}_kb_$1.log 2>&1
done
timeout 900 python scripts/profile_cost.py --reps 3 > gpurun_out/${TAG}_profile_cost.jsonl 2> gpurun_out/${TAG}_profile_cost.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for f in gpurun_out/${TAG}_*.log gpurun_out/${TAG}_*.jsonl; do echo "== $f"; tail -n 12 "$f" | cut -c1-400; done

TAG=${1:-r02h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "shared_queue or tiled or gemm_full or stress" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1500 python scripts/search_sweep.py --nt auto --spaces b200:coulomb,b200:transpose,b200:gemm --runs 5 --mq "off;4,1,4;8,2,4;8,3,4;12,3,4;12,4,4;16,4,4" > gpurun_out/${TAG}_mq_sweep.jsonl 2> gpurun_out/${TAG}_mq_sweep.err; echo "rc=$?" >> gpurun_out/${TAG}_mq_sweep.err
timeout 1500 python scripts/search_sweep.py --nt auto --spaces gemm_full,stress:1048576,stress:4194304 --reps 444 --outer 10 --runs 2 --env "CT_SEARCH_TILED=0;CT_SEARCH_TILED=1" > gpurun_out/${TAG}_tiled_sweep.jsonl 2> gpurun_out/${TAG}_tiled_sweep.err; echo "rc=$?" >> gpurun_out/${TAG}_tiled_sweep.err
for f in gpurun_out/${TAG}_*; do echo "== $f"; tail -n 30 "$f" | cut -c1-400; done

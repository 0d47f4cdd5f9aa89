TAG=${1:-q}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for pre in 1 0; do echo "== PRE=$pre"; CT_SEARCH_PRE=$pre timeout 300 python bench.py --steps 10 --warmup 3 --kernel-only 2>&1 | grep "\[bench\]"; done > gpurun_out/${TAG}_timing.log
tail -n 4 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_timing.log

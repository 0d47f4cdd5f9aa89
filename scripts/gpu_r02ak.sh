TAG=${1:-r02ak}
mkdir -p gpurun_out
timeout 1500 python scripts/live_experiment.py datasets/gemm-b200 datasets/conv-b200 --live 10 --measured-overhead --out gpurun_out/${TAG}_live_full.json > gpurun_out/${TAG}_live_full.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_full.log
timeout 1500 python scripts/live_experiment.py datasets/gemm-b200 datasets/conv-b200 --live 10 --mode group1 --measured-overhead --out gpurun_out/${TAG}_live_group1.json > gpurun_out/${TAG}_live_group1.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_group1.log
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-200; done

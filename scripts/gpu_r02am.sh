# conv live searches with cold compiles (the r02al call ran out of time before conv)
TAG=${1:-r02am}
mkdir -p gpurun_out
export CUDA_CACHE_DISABLE=1
timeout 780 python scripts/live_experiment.py datasets/conv-b200 --live 6 --measured-overhead > gpurun_out/${TAG}_live_full.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_full.log
timeout 600 python scripts/live_experiment.py datasets/conv-b200 --live 6 --mode group1 --measured-overhead > gpurun_out/${TAG}_live_group1.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_group1.log

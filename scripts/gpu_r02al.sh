# Live searches with the driver's compute cache disabled: every search
# compiles and loads its variants cold, as a fresh tuning session does
# (r02ak and earlier ran with ~/.nv/ComputeCache warm from earlier searches
# of the same process or box, scripts/debug/compile_cache.py).
TAG=${1:-r02al}
mkdir -p gpurun_out
export CUDA_CACHE_DISABLE=1
for s in 1 1; do python scripts/debug/compile_cache.py datasets/gemm-b200 gemm $s; done > gpurun_out/${TAG}_cache_probe.log 2>&1
D="datasets/coulomb-b200 datasets/nbody-b200 datasets/transpose-b200 datasets/gemm-b200 datasets/conv-b200"
timeout 1700 python scripts/live_experiment.py $D --live 10 --measured-overhead --out gpurun_out/${TAG}_live_full.json > gpurun_out/${TAG}_live_full.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_full.log
timeout 1500 python scripts/live_experiment.py $D --live 10 --mode group1 --measured-overhead --out gpurun_out/${TAG}_live_group1.json > gpurun_out/${TAG}_live_group1.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_live_group1.log
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-200; done

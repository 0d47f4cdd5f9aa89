TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 300 python scripts/debug/cupti_dram.py > gpurun_out/${TAG}_cupti_dram.log 2>&1
timeout 900 python scripts/debug/conv_cases.py 1024 256 0,33,360,978,1449,2354,2966,3191,3439,3924,3927 > gpurun_out/${TAG}_conv_cases.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python bench.py --steps 1 --warmup 3 --kernel-only --no-cpu-baseline > gpurun_out/${TAG}_clk.log 2>&1
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 6 "$f" | cut -c1-600; done

# shared-queue search kernel: parity on every trajectory set, then timings of
# every build against k_profile_search on the five B200 spaces
TAG=${1:-r02f}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "shared_queue" > gpurun_out/${TAG}_pytest_mq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_mq.log
timeout 1500 python scripts/search_sweep.py --nt auto --spaces b200:coulomb,b200:transpose,b200:nbody,b200:conv,b200:gemm --runs 5 --mq "off;4,1,4;6,2,4;8,2,4;8,3,4;12,3,4;12,4,4;16,4,4" > gpurun_out/${TAG}_mq_sweep.jsonl 2> gpurun_out/${TAG}_mq_sweep.err; echo "rc=$?" >> gpurun_out/${TAG}_mq_sweep.err
timeout 900 python -X faulthandler scripts/debug/cupti_switch.py > gpurun_out/${TAG}_cupti_switch.log 2>&1
for f in gpurun_out/${TAG}_*; do echo "== $f"; tail -n 50 "$f" | cut -c1-300; done

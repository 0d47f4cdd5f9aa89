# search kernel variants: parity under each, timing, phase clocks
# usage: bash scripts/ws_experiment.sh <tag>
TAG=${1:-ws}
mkdir -p gpurun_out
{
for ws in 0 2 3 4 6 8; do
  echo "== CT_SEARCH_WS=$ws"
  CT_SEARCH_WS=$ws timeout 300 python bench.py --steps 10 --warmup 3 --kernel-only 2>&1 | grep "\[bench\]"
done
for ws in 0 4; do
  echo "== clocks CT_SEARCH_WS=$ws"
  CT_SEARCH_WS=$ws CT_LIB_PATH=paper_2102_05297_b200/libct_b200_clk.so timeout 300 python bench.py --steps 1 --warmup 3 --kernel-only 2>&1 | grep -E "clk" | head -12
done
} > gpurun_out/${TAG}_timing.log 2>&1
for ws in 0 4; do
  CT_SEARCH_WS=$ws timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_ws$ws.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_ws$ws.log
done
tail -n 3 gpurun_out/${TAG}_pytest_ws*.log; cat gpurun_out/${TAG}_timing.log

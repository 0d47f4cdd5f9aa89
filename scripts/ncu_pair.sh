# ncu --set full of the search kernel under two kernel variants
TAG=${1:-pair}
mkdir -p gpurun_out
for ws in 0 6; do
  CT_SEARCH_WS=$ws timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_profile_search -c 1 -o gpurun_out/${TAG}_ws$ws python bench.py --steps 1 --warmup 3 --kernel-only > gpurun_out/${TAG}_ws$ws.log 2>&1
done
ls -la gpurun_out/${TAG}_*

# ncu --set full of the best configuration of every B200 sweep
mkdir -p gpurun_out
for b in transpose coulomb nbody conv gemm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${b}\$" -s 1 -c 1 \
      -o gpurun_out/kb_${b} python scripts/run_variant.py --bench $b --best datasets/${b}-b200 \
      > gpurun_out/kb_${b}.log 2>&1
  tail -n 2 gpurun_out/kb_${b}.log
done
ls -la gpurun_out/kb_*

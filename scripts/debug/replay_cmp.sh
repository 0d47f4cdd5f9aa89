for b in transpose coulomb gemm nbody conv; do
  CT_TUNE_REPLAY=user timeout 300 python scripts/debug/replay_values.py $b > gpurun_out/r02n_vals_user_$b.json 2> gpurun_out/r02n_vals_user_$b.err
  CT_TUNE_REPLAY=kernel timeout 300 python scripts/debug/replay_values.py $b > gpurun_out/r02n_vals_kernel_$b.json 2> gpurun_out/r02n_vals_kernel_$b.err
done
python - <<'PY'
import json
for b in ["transpose","coulomb","gemm","nbody","conv"]:
    try:
        u=json.load(open(f"gpurun_out/r02n_vals_user_{b}.json")); k=json.load(open(f"gpurun_out/r02n_vals_kernel_{b}.json"))
    except Exception as e:
        print(b, "missing", e); continue
    print("==", b, "passes user", u["passes"], "kernel", k["passes"])
    for a in u["run0"]:
        x,y=u["run0"][a],k["run0"].get(a)
        print(f"  {a:14s} user {x:16.6g} kernel {y:16.6g} rel {abs(x-y)/max(abs(x),1e-9):.3g}")
PY

for b in transpose coulomb; do
  timeout 300 python scripts/debug/replay_values.py $b > gpurun_out/r02o_vals_set_$b.json 2> gpurun_out/r02o_vals_set_$b.err
  CT_TUNE_KEEP_CONFIG=1 timeout 300 python scripts/debug/replay_values.py $b > gpurun_out/r02o_vals_keep_$b.json 2> gpurun_out/r02o_vals_keep_$b.err
  CT_TUNE_KEEP_CONFIG=1 CT_TUNE_TRACE=1 timeout 300 python scripts/profile_cost.py --one $b:steps --reps 3 > gpurun_out/r02o_keep_steps_$b.log 2>&1
done
python - <<'PY'
import json
for b in ["transpose","coulomb"]:
    u=json.load(open(f"gpurun_out/r02o_vals_set_{b}.json")); k=json.load(open(f"gpurun_out/r02o_vals_keep_{b}.json"))
    print("==", b, "passes", u["passes"], k["passes"])
    for run in ("run0", "run1"):
        bad=[(a,u[run][a],k[run][a]) for a in u[run] if abs(u[run][a]-k[run][a])>0.02*max(abs(u[run][a]),1)]
        print(run, "differ:", bad[:8])
PY
tail -3 gpurun_out/r02o_keep_steps_*.log | cut -c1-600

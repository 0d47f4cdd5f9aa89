"""Markdown table of the cross-input improvement matrix (scripts/cross_matrix.py
JSON): rows = run dataset, columns = model dataset, cells = improvement of the
profile searcher over random search (mean empirical steps to <= 1.1x best)."""
import json
import sys

d = json.load(open(sys.argv[1]))
fams = {}
for v in d.values():
    fams.setdefault(v["run"].split("-")[0], {}).setdefault(v["run"], {})[v["model"]] = v
for fam, runs in fams.items():
    models = sorted({m for r in runs.values() for m in r}, key=lambda x: (x != fam, x))
    print(f"\n{fam} family (rows: run on, columns: model from; improvement over random search)\n")
    print("| run \\ model | " + " | ".join(models) + " | random steps |")
    print("|---" * (len(models) + 2) + "|")
    for run in sorted(runs, key=lambda x: (x != fam, x)):
        cells = []
        for m in models:
            v = runs[run].get(m)
            cells.append("—" if v is None else f"{v['improvement']:.2f}× ({v['profile_mean_steps']:.1f})")
        rnd = next(iter(runs[run].values()))["random_mean_steps"]
        print(f"| {run} ({next(iter(runs[run].values()))['configs']}) | " + " | ".join(cells) + f" | {rnd:.1f} |")

"""Time the batched search kernel on every synthetic space for several CTA
sizes (CT_SEARCH_NT).  GPU only; CUDA events on the context's stream.

    python scripts/search_sweep.py [--nt 32,64,128] [--spaces coulomb,transpose]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nt", default="32,64,128,256,512")
    ap.add_argument("--spaces", default="coulomb,transpose,nbody,conv,gemm")
    ap.add_argument("--reps", type=int, default=1000)
    ap.add_argument("--outer", type=int, default=40)
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--kernel-only", action="store_true", help="one launch per space (ncu)")
    ap.add_argument("--env", default="",
                    help="';'-separated environment variants, each 'K=V+K=V' (e.g. CT_SEARCH_TILED=1)")
    a = ap.parse_args()
    import torch
    from paper_2102_05297_b200 import ExactModelSet, harness, spaces
    from paper_2102_05297_b200 import _native
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _native.context(0)
    ctx.set_stream(stream.cuda_stream)
    from paper_2102_05297_b200 import formats
    hbm = 6548.5
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
    except Exception:
        pass
    for name in a.spaces.split(","):
        # "<name>" = synthetic stand-in, "b200:<name>" = datasets/<name>-b200
        if name.startswith("b200:"):
            ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", name[5:] + "-b200"))
        elif name.startswith("stress:"):
            # BASELINE.md section 3 stress sizes: the table exceeds the L2
            ds = spaces.stress(int(name[7:]))
        else:
            ds = spaces.SPACES[name]()
        spec = harness.ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                      repetitions=a.reps, outer_iterations=a.outer, seed=42,
                                      stop_at_well_performing=False)
        params, _ = harness.prepare_device(ctx, spec)
        ref = None
        envs = a.env.split(";") if a.env else [""]
        for nt, ev in [(x, z) for z in envs for x in a.nt.split(",")]:
            for kv in [k for k in (a.env.replace(";", "+").split("+") if a.env else []) if k]:
                os.environ.pop(kv.split("=")[0], None)
            for kv in [k for k in ev.split("+") if k]:
                key, val = kv.split("=")
                os.environ[key] = val
            if nt == "auto":
                os.environ.pop("CT_SEARCH_NT", None)     # the launcher's choice
            else:
                os.environ["CT_SEARCH_NT"] = nt
            harness.launch(ctx, spec, params, 0, a.reps)   # warm-up
            times = []
            for _ in range(0 if a.kernel_only else a.runs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                harness.launch(ctx, spec, params, 0, a.reps)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            idx, _, nst, _, _, stats = ctx.fetch(a.reps, want_profiled=False)
            same = None
            if ref is None:
                ref = (idx.copy(), nst.copy())
            else:
                same = bool((ref[1] == nst).all() and (ref[0] == idx).all())
            if a.kernel_only:
                continue
            ms = sorted(times)[len(times) // 2]
            gbs = stats.algorithmic_bytes / (ms / 1e3) / 1e9
            print(json.dumps({"space": name, "n": len(ds.space), "nt": nt, "env": ev, "ms": ms,
                              "reps": a.reps, "outer": a.outer,
                              "algorithmic_bytes": int(stats.algorithmic_bytes),
                              "configs_per_s": stats.configs_scored / (ms / 1e3),
                              "algorithmic_GBps": gbs, "hbm_frac": gbs / hbm,
                              "uncertified": int(stats.uncertified),
                              "same_as_first": same}), flush=True)
    os.environ.pop("CT_SEARCH_NT", None)


if __name__ == "__main__":
    main()

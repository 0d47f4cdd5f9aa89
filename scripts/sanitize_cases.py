"""Small invocations of every device path for compute-sanitizer
(scripts/sanitize.sh): python scripts/sanitize_cases.py <case>

  scratch   b200 gemm, weights in a global slice (CT_SEARCH_SMEM=0)
  ws        warp-specialised two-repetition kernel (CT_SEARCH_WS=4)
  hg        400,000-configuration stress space: row index in global scratch
  topk      score_top_k on b200 transpose
  report    simulate() with the one-call device report
  tune      libct_tune: compile, time and profile one transpose variant
  tiled     the tiled large-space path (CT_SEARCH_TILED=1) on b200 gemm
  seq       every draw through the warp's binade-exact sequential re-decision
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def search(ds, **kw):
    from paper_2102_05297_b200 import ExactModelSet, harness
    spec = harness.ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                  repetitions=kw.pop("reps", 6), outer_iterations=kw.pop("i", 4),
                                  seed=5, **kw)
    res, _ = harness.run_batch(spec)
    print("steps", res.n_steps.tolist(), "uncertified", res.uncertified)


def main():
    case = sys.argv[1]
    from paper_2102_05297_b200 import formats, spaces
    b200 = lambda n: formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{n}-b200"))
    if case == "scratch":
        os.environ["CT_SEARCH_SMEM"] = "0"
        search(b200("gemm"))
    elif case == "ws":
        os.environ["CT_SEARCH_WS"] = "4"
        search(b200("transpose"))
    elif case == "hg":
        search(spaces.stress(400_000), reps=2, i=3, stop_at_well_performing=False)
    elif case == "tiled":
        os.environ["CT_SEARCH_TILED"] = "1"
        search(b200("gemm"))
    elif case == "seq":
        os.environ["CT_SEARCH_FORCE_SEQUENTIAL"] = "1"
        search(b200("transpose"))
    elif case == "topk":
        search(b200("transpose"), score_top_k=40)
    elif case == "report":
        from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, simulate
        ds = b200("coulomb")
        rep = simulate(ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                      repetitions=16, seed=3, time_repetitions=8))
        print("mean steps", rep.mean_steps)
    elif case == "tune":
        from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
        src = CudaMeasurementSource(benchmark("transpose", width=1024, height=1024))
        m = src.measure(0, profiled=False)     # CUPTI cannot run under the sanitizer
        print("runtime", m.runtime_us)
        src.close()
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main()

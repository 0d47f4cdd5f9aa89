"""Record dataset-format fixtures with the reference itself (build container
only: imports /root/reference/pkg/src).  Writes tests/golden/formats/:

  ref_volta/      save_dataset() of a 60-configuration volta_plus dataset
                  (arch with a map./ratio. override)
  ref_prevolta/   the same space measured under pre-Volta counter names,
                  written as raw names (load path canonicalises them)
  raw_volta.csv   a measurements file with raw Volta+ metric names
  expect.npz      what the reference's loader returns for each of them

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_formats_golden.py
"""

import os
import shutil

import numpy as np
from countertune import counters, space

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")


def build(generation, raw_names):
    params = (space.TuningParameter.make("BLOCK", [32, 64, 128, 256]),
              space.TuningParameter.make("VEC", [1, 2, 4]),
              space.TuningParameter.make("SMEM", [0, 1]),
              space.TuningParameter.make("TILE", [0.5, 1.25, 3.0]))
    grid = [(b, v, s, t) for b in params[0].values for v in params[1].values
            for s in params[2].values for t in params[3].values][:60]
    confs = tuple(space.TuningConfiguration(assignment=tuple(map(float, g)), index=i)
                  for i, g in enumerate(grid))
    sp = space.TuningSpace(parameters=params, configurations=confs)
    arch = counters.ArchProfile(name=f"test-{generation}", generation=generation, cores=2944,
                                overrides={"my_fancy_dram_ctr": ("DRAM_RT", 0.5)})
    rng = np.random.default_rng(11)
    recs = []
    for i in range(len(sp)):
        cmap = {}
        for d in counters.CATALOG:
            if d.abbr == counters.GLOBAL_THREADS:
                continue
            lo, hi = counters.VALUE_RANGES[d.abbr]
            cmap[d.abbr] = float(rng.uniform(0, hi if hi else 1e7))
        recs.append(space.MeasurementRecord(config_index=i,
                                            runtime_us=float(rng.uniform(1, 1000)),
                                            global_threads=int(rng.integers(1, 1 << 20)),
                                            counters=cmap))
    return space.Dataset(space=sp, arch=arch, input_label="x", records=tuple(recs))


def main():
    if os.path.isdir(HERE):
        shutil.rmtree(HERE)
    os.makedirs(HERE)
    expect = {}
    for gen in ("volta_plus", "pre_volta"):
        ds = build(gen, raw_names=False)
        d = os.path.join(HERE, f"ref_{gen}")
        space.save_dataset(ds, d)
        back = space.load_dataset_dir(d)
        names = back.counter_names
        expect[f"{gen}_names"] = np.array(names)
        expect[f"{gen}_runtime"] = np.array([r.runtime_us for r in back.records])
        expect[f"{gen}_threads"] = np.array([r.global_threads for r in back.records])
        expect[f"{gen}_matrix"] = np.array([[r.counters[a] for a in names] for r in back.records])
        expect[f"{gen}_assign"] = np.array([c.assignment for c in back.space.configurations])
    # raw Volta+ metric names plus the arch override column: loader canonicalises
    ds = build("volta_plus", raw_names=True)
    cols = []
    for d in counters.CATALOG:
        if d.abbr in (counters.GLOBAL_THREADS, "DRAM_RT"):
            continue
        cols.append((d.volta_name, d.abbr, d.volta_scale))
    lines = ["config_index,runtime_us,global_threads,my_fancy_dram_ctr,"
             + ",".join(c[0] for c in cols)]
    for r in ds.records:
        cells = [str(r.config_index), repr(r.runtime_us), str(r.global_threads),
                 repr(r.counters["DRAM_RT"] * 2.0)]
        cells += [repr(r.counters[a] / s) for _, a, s in cols]
        lines.append(",".join(cells))
    raw_dir = os.path.join(HERE, "raw_volta")
    os.makedirs(raw_dir)
    shutil.copy(os.path.join(HERE, "ref_volta_plus", "space.csv"), raw_dir)
    shutil.copy(os.path.join(HERE, "ref_volta_plus", "arch.txt"), raw_dir)
    with open(os.path.join(raw_dir, "measurements.csv"), "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
    back = space.load_dataset_dir(raw_dir)
    names = back.counter_names
    expect["raw_names"] = np.array(names)
    expect["raw_matrix"] = np.array([[r.counters[a] for a in names] for r in back.records])
    np.savez(os.path.join(HERE, "expect.npz"), **expect)
    print("wrote", HERE)


if __name__ == "__main__":
    main()

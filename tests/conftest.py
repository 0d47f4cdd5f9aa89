import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def ragged(traj, key):
    """Split a flattened trajectory set into per-repetition lists."""
    idx = traj[key + "_idx"]
    off = traj[key + "_off"]
    return [idx[off[r]:off[r + 1]].tolist() for r in range(off.size - 1)]


def dataset_from_golden(name):
    """Our Dataset built from a recorded ds_<name>.npz (no reference needed)."""
    from paper_2102_05297_b200.counters import ArchProfile
    from paper_2102_05297_b200.space import Dataset, TuningParameter, TuningSpace
    d = golden(f"ds_{name}.npz")
    params = []
    for pname, binary, j in zip(d["param_names"], d["param_binary"], range(len(d["param_names"]))):
        vals = tuple(sorted(set(d["assignments"][:, j].tolist())))
        params.append(TuningParameter(name=str(pname), values=vals, is_binary=bool(binary)))
    space = TuningSpace.from_assignments(params, d["assignments"])
    gen = "pre_volta" if int(d["generation"]) == 0 else "volta_plus"
    arch = ArchProfile(name=str(d["arch_name"]), generation=gen, cores=int(d["cores"]))
    return Dataset(space, arch, str(d["input_label"]), runtime_us=d["runtime"],
                   global_threads=d["threads"],
                   counter_names=tuple(str(x) for x in d["counter_names"]),
                   counter_matrix=d["counter_matrix"])


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def hostcheck():
    import ctypes
    path = os.path.join(ROOT, "tests", "native", "_hostcheck.so")
    if not os.path.exists(path):
        import __graft_entry__
        __graft_entry__.build_hostcheck()
    return ctypes.CDLL(path)

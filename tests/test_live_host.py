"""Host-side logic of the live measurement path (no GPU): spaces match Table 2
of the paper and the synthetic stand-ins, variant options, launch geometry
and argument packing, and the tuner library's error behaviour without a
device."""

import ctypes
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT, have_gpu

TABLE2 = {"coulomb": 210, "transpose": 1784, "nbody": 3134, "conv": 3928, "gemm": 5788}


@pytest.mark.parametrize("name", sorted(TABLE2))
def test_space_sizes_and_identity_with_synthetic(name):
    from paper_2102_05297_b200 import live, spaces
    b = live.benchmark(name)
    assert len(b.space) == TABLE2[name]
    ds = spaces.SPACES[name]()
    assert np.array_equal(b.space.assignments, ds.space.assignments)
    assert b.space.parameter_names == ds.space.parameter_names


def test_gemm_full_space_size():
    from paper_2102_05297_b200 import spaces
    assert len(spaces.space_of("gemm_full")) == 205216


def test_launch_packing():
    from paper_2102_05297_b200.tuner import Launch
    l = Launch((4, 2), (32,), [ctypes.c_uint64(0x1234), ctypes.c_int32(7), ctypes.c_float(1.5),
                               ctypes.c_uint64(9)])
    assert tuple(l.c.grid) == (4, 2, 1) and tuple(l.c.block) == (32, 1, 1)
    offs = [l.c.arg_offsets[i] for i in range(l.c.n_args)]
    assert offs == [0, 8, 12, 16]
    raw = ctypes.string_at(l.c.args, 24)
    assert int.from_bytes(raw[0:8], "little") == 0x1234
    assert int.from_bytes(raw[8:12], "little") == 7
    assert np.frombuffer(raw[12:16], np.float32)[0] == 1.5
    assert l.threads == 4 * 2 * 32


@pytest.mark.parametrize("name", sorted(TABLE2))
def test_launch_geometry_covers_problem(name):
    """Every configuration's grid x per-block work covers the problem exactly
    and the block fits the 1024-thread limit."""
    from paper_2102_05297_b200 import live
    b = live.benchmark(name)
    bufs = {k: 0 for k in ("in", "out", "atoms", "x", "y", "z", "w", "energy", "pm", "m",
                           "acc", "filt", "at", "b", "c", "partial", "arrivals")}
    if name == "gemm":      # TMA descriptors need a device context; geometry does not
        b.tensor_maps = lambda v, bufs: ()
    for i in range(len(b.space)):
        v = b.values(i)
        l = b.launch(v, bufs)
        assert np.prod(l.block) <= 1024
        if name == "transpose":
            assert l.grid[0] * v["TILE"] * v["WORK_X"] == b.width
            assert l.grid[1] * v["TILE"] == b.height
        elif name == "coulomb":
            assert l.grid[0] * 32 == b.grid and l.grid[1] * l.block[1] == b.grid
            assert l.grid[2] * v["Z_ITERATIONS"] >= b.grid
        elif name == "nbody":
            assert l.grid[0] * v["BLOCK"] * v["OUTER"] >= b.bodies
            assert 1 <= l.grid[1] <= b.MAX_JB and l.block[0] * l.block[1] <= 1024
            # the j range splits evenly enough that no thread row is idle
            splits = l.grid[1] * l.block[1]
            tiles = -(-b.bodies // v["BLOCK"])
            assert -(-tiles // splits) * (splits - 1) < tiles
        elif name == "conv":
            assert l.grid[0] * v["TBX"] * v["WPTX"] == b.width
            assert l.grid[1] * v["TBY"] * v["WPTY"] == b.height
            assert l.c.dynamic_smem <= 227 * 1024
        elif name == "gemm":
            assert l.grid[0] * v["MWG"] == b.m and l.grid[1] * v["NWG"] == b.n


@pytest.mark.parametrize("name", sorted(TABLE2))
def test_sample_variants_compile_for_sm100a(name, tmp_path):
    """A seeded sample of each space compiles offline for sm_100a (nvcc on the
    NVRTC source with the variant's -D options)."""
    from paper_2102_05297_b200 import live
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc missing")
    b = live.benchmark(name)
    src = os.path.join(ROOT, "paper_2102_05297_b200", "kernels", b.kernel + ".cu")
    rng = np.random.default_rng(7)
    for i in sorted(set(rng.choice(len(b.space), 3, replace=False).tolist())):
        r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-cubin",
                            "-std=c++17", "-o", str(tmp_path / "v.cubin"), *b.options(b.values(i)),
                            src], capture_output=True, text=True)
        assert r.returncode == 0, (i, b.values(i), r.stderr[-2000:])


def test_tuner_without_gpu_fails_loudly():
    if have_gpu():
        pytest.skip("a GPU is present")
    from paper_2102_05297_b200.errors import CounterTuneError
    from paper_2102_05297_b200.tuner import Tuner
    with pytest.raises(CounterTuneError, match="no CUDA device"):
        Tuner(0)


def test_table1_metric_set():
    from paper_2102_05297_b200 import counters as cc
    from paper_2102_05297_b200.live import TABLE1_ABBRS, TABLE1_METRICS
    assert len(TABLE1_METRICS) == 24 and len(set(TABLE1_METRICS)) == 24
    assert set(cc.REQUIRED_COUNTERS) <= set(TABLE1_ABBRS)

"""The device arithmetic (csrc/*.cuh), compiled for the host, against the
reference's fixtures and numpy -- runs without a GPU.

tests/native/_hostcheck.so is a test-only build of the same headers the
kernels include (RNG, expert system, pow8, Eq. 17 weight, exact fixed point,
certified selection and a sequential replay of the kernel's per-repetition
algorithm).  This pins the device code paths before they reach a B200.
"""

import ctypes
from fractions import Fraction

import numpy as np
import pytest

from conftest import golden, ragged

P = ctypes.POINTER
dp = P(ctypes.c_double)


def a_(x, t):
    return x.ctypes.data_as(P(t))


def words(v):
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & 0xFFFFFFFF)
        v >>= 32
    return out


def test_seed_sequence_pool_and_streams(hostcheck):
    for seed in (0, 42, 7, 2 ** 70 + 3):
        ent = np.array(words(seed), dtype=np.uint32)
        pre = np.zeros(1, dtype=np.uint32)
        children = np.random.SeedSequence(seed).spawn(24)
        for r, ch in enumerate(children):
            out = np.zeros(4, dtype=np.uint32)
            hostcheck.hc_seed_pool(a_(ent, ctypes.c_uint32), len(ent), a_(pre, ctypes.c_uint32), 0,
                                   1, ctypes.c_uint32(r), a_(out, ctypes.c_uint32))
            assert out.tolist() == [int(v) for v in ch.pool]
            g = np.random.default_rng(ch)
            ops = np.array([0] + [1] * 20 + [0, 0, 1, 0], dtype=np.int32)
            args = np.array([1784] + [0] * 20 + [7, 1, 0, 205216], dtype=np.int64)
            want = ([g.integers(0, 1784)] + list(g.random(20)) +
                    [g.integers(0, 7), g.integers(0, 1), g.random(), g.integers(0, 205216)])
            got = np.zeros(len(ops))
            hostcheck.hc_rng_stream(a_(ent, ctypes.c_uint32), len(ent), a_(pre, ctypes.c_uint32),
                                    0, 1, ctypes.c_uint32(r), a_(ops, ctypes.c_int),
                                    a_(args, ctypes.c_int64), len(ops), a_(got, ctypes.c_double))
            assert got.tolist() == [float(v) for v in want]
            perm = np.zeros(997, dtype=np.int64)
            hostcheck.hc_permutation(a_(ent, ctypes.c_uint32), len(ent), a_(pre, ctypes.c_uint32), 0,
                                     1, ctypes.c_uint32(r), ctypes.c_int64(997),
                                     a_(perm, ctypes.c_int64))
            assert perm.tolist() == np.random.default_rng(ch).permutation(997).tolist()


def test_expert_system_bit_exact(hostcheck):
    e = golden("expert.npz")
    for k in range(e["counters"].shape[0]):
        c = np.ascontiguousarray(e["counters"][k])
        b = np.zeros(18)
        d = np.zeros(18)
        deg = hostcheck.hc_analyze(a_(c, ctypes.c_double), int(e["generation"][k]),
                                   ctypes.c_int64(int(e["cores"][k])),
                                   ctypes.c_int64(int(e["threads"][k])), a_(b, ctypes.c_double))
        hostcheck.hc_react(a_(b, ctypes.c_double), ctypes.c_double(float(e["inst_reaction"][k])),
                           ctypes.c_double(-1.0), a_(d, ctypes.c_double))
        np.testing.assert_array_equal(b.view(np.uint64), e["b"][k].view(np.uint64))
        np.testing.assert_array_equal(d.view(np.uint64), e["delta"][k].view(np.uint64))
        assert bool(deg) == bool(e["degenerate"][k])


def test_pow8_correctly_rounded(hostcheck):
    rng = np.random.default_rng(3)
    x = np.concatenate([1 + rng.random(3000), rng.random(3000), np.array([0.0, 1.0, 2.0, 0.5])])
    out = np.zeros_like(x)
    hostcheck.hc_pow8(a_(x, ctypes.c_double), ctypes.c_int64(x.size), a_(out, ctypes.c_double))
    for xi, oi in zip(x, out):
        assert float(Fraction(xi) ** 8) == oi      # float(Fraction) rounds correctly
    # numpy's pow (SVML or glibc) is within 1 ulp of it
    assert np.abs((x ** 8).view(np.int64) - out.view(np.int64)).max() <= 1


def test_weights_within_one_ulp_of_reference(hostcheck):
    s = golden("scores.npz")
    for k in range(int(s["cases"])):
        raw = s[f"raw_{k}"]
        explored = s[f"explored_{k}"].astype(bool)
        scoreable = s[f"scoreable_{k}"]
        pool = ~explored if scoreable.size == 0 else (scoreable.astype(bool) & ~explored)
        pool_u8 = pool.astype(np.uint8)
        out = np.zeros_like(raw)
        hostcheck.hc_weights(a_(raw, ctypes.c_double), a_(pool_u8, ctypes.c_uint8),
                             ctypes.c_int64(raw.size), ctypes.c_double(float(raw[pool].max())),
                             ctypes.c_double(float(raw[pool].min())), ctypes.c_double(-0.25),
                             a_(out, ctypes.c_double))
        assert np.abs(out.view(np.int64) - s[f"norm_{k}"].view(np.int64)).max() <= 1


def test_fixed_point_is_exact(hostcheck):
    rng = np.random.default_rng(9)
    w = np.concatenate([rng.uniform(1e-4, 256.0, 5000), [1e-4, 256.0, 1.0, 0.0, 3.5]])
    back = np.zeros_like(w)
    fl = np.zeros_like(w)
    ok = hostcheck.hc_fx_roundtrip(a_(w, ctypes.c_double), ctypes.c_int64(w.size),
                                   a_(back, ctypes.c_double), a_(fl, ctypes.c_double))
    assert ok == 1
    np.testing.assert_array_equal(back, w)
    np.testing.assert_array_equal(fl, w)
    hostcheck.hc_fx_sum.restype = ctypes.c_double
    total = hostcheck.hc_fx_sum(a_(w, ctypes.c_double), ctypes.c_int64(w.size))
    assert total == float(sum(Fraction(v) for v in w))


def test_certified_selection_matches_numpy(hostcheck):
    hostcheck.hc_select.restype = ctypes.c_int64
    rng = np.random.default_rng(21)
    uncertified = 0
    for _ in range(400):
        n = int(rng.integers(1, 3000))
        w = np.where(rng.random(n) < 0.5, rng.uniform(1.0, 256.0, n), rng.uniform(1e-4, 1.0, n))
        w[rng.random(n) < 0.2] = 0.0
        if not w.any():
            w[-1] = 1.0
        u = rng.random()
        c = np.cumsum(w)
        want = int(np.searchsorted(c, u * c[-1], side="right"))
        cert = ctypes.c_int(0)
        got = hostcheck.hc_select(a_(w, ctypes.c_double), ctypes.c_int64(n), ctypes.c_double(u),
                                  ctypes.byref(cert))
        assert got == want
        uncertified += cert.value == 0
    assert uncertified < 5


class _Params(ctypes.Structure):
    _fields_ = [("outer_iterations", ctypes.c_int32), ("inner_steps", ctypes.c_int32),
                ("inst_reaction", ctypes.c_double), ("issue_delta_sign", ctypes.c_double),
                ("gamma", ctypes.c_double), ("literal_sign", ctypes.c_int32),
                ("score_top_k", ctypes.c_int64), ("use_stop", ctypes.c_int32),
                ("generation", ctypes.c_int32), ("cores", ctypes.c_int64),
                ("delta_columns", ctypes.c_int32 * 18)]


@pytest.mark.parametrize("name", ["gradient", "calibration", "transpose", "coulomb"])
def test_kernel_algorithm_reproduces_reference_trajectories(hostcheck, name):
    """The kernel's per-repetition algorithm (exact prefix + certification +
    device RNG), run sequentially on the host, against reference trajectories."""
    from paper_2102_05297_b200.counters import DELTA_KEYS
    d = golden(f"ds_{name}.npz")
    traj = golden(f"traj_{name}.npz")
    reps, i = int(traj["reps"]), int(traj["i"])
    n = d["runtime"].size
    stop = np.zeros(n, dtype=np.uint8)
    stop[traj["well"]] = 1
    hr = np.ones(n, dtype=np.uint8)
    keys = sorted({k[:-4] for k in traj.files if k.endswith("_idx") and not k.startswith("random")})
    ent = np.array([42], dtype=np.uint32)
    pre = np.zeros(1, dtype=np.uint32)
    req = np.ascontiguousarray(d["required"])
    thr = np.ascontiguousarray(d["threads"].astype(np.int64))
    rt = np.ascontiguousarray(d["runtime"])
    for key in keys:
        model = key.split("_")[0]
        names = [str(x) for x in d[f"{model}_names"]]
        table = np.ascontiguousarray(d[f"{model}_matrix"].T)
        prm = _Params(outer_iterations=i, inner_steps=5, inst_reaction=0.7, issue_delta_sign=-1.0,
                      gamma=-0.25, literal_sign=int(key.endswith("_literal")), score_top_k=-1,
                      use_stop=int("_stop" in key), generation=int(d["generation"]),
                      cores=int(d["cores"]))
        for k, dk in enumerate(DELTA_KEYS):
            prm.delta_columns[k] = names.index(dk) if dk in names else -1
        want = ragged(traj, key)
        for r in range(reps):
            oi = np.zeros(i * 6, dtype=np.int32)
            op = np.zeros(i * 6, dtype=np.uint8)
            ns, unc, sc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            hostcheck.hc_profile_search(
                a_(table, ctypes.c_double), ctypes.c_int64(n), a_(rt, ctypes.c_double),
                a_(thr, ctypes.c_int64), a_(req, ctypes.c_double), a_(hr, ctypes.c_uint8),
                a_(stop, ctypes.c_uint8) if "_stop" in key else None, ctypes.byref(prm),
                a_(ent, ctypes.c_uint32), 1, a_(pre, ctypes.c_uint32), 0, 1, ctypes.c_uint32(r),
                a_(oi, ctypes.c_int32), a_(op, ctypes.c_uint8), ctypes.byref(ns),
                ctypes.byref(unc), ctypes.byref(sc))
            assert oi[:ns.value].tolist() == want[r], (key, r)
            assert unc.value == 0

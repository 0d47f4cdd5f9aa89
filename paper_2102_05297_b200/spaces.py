"""Synthetic replay datasets shaped like the paper's five benchmark spaces.

Real exhaustive B200 sweeps need the live NVRTC launcher + CUPTI collector
(not built yet).  Until they exist, the searcher
is exercised on closed-form stand-ins: each space enumerates its tuning
parameters under the kernel's launch constraints, is cut to the size Table 2
of the paper gives by a seeded subsample when the
constraint set leaves more, and gets all 24 Table-1 counters plus runtime from
one analytic B200 model (bandwidth / pipe / issue / occupancy terms).  Every
value is a deterministic function of the parameters, so datasets are
reproducible byte for byte.

    coulomb    210 configs,   7 params  (Coulomb sum 256^3 grid, 256 atoms)
    transpose  1,784 configs, 8 params  (8192^2 fp32)
    nbody      3,134 configs, 7 params  (16,384 bodies)
    conv       3,928 configs, 10 params (4096^2, 7x7 filter)
    gemm       5,788 configs, 10 params (2048^3 sgemm, CLBlast-style)
    gemm_full  205,216 configs, 14 params
    stress(n)  n configs (BASELINE.md section 3 stress sizes 1,048,576 and
               4,194,304): random counters, the scoring microbenchmark's table
"""

import itertools
from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

from .counters import ArchProfile, REQUIRED_COUNTERS
from .space import Dataset, TuningParameter, TuningSpace

B200_SMS = 148
B200_CORES = B200_SMS * 128
B200_ARCH = ArchProfile(name="b200", generation="volta_plus", cores=B200_CORES)

_CLOCK = 1.9e9
_HBM = 6.55e12          # B/s, MEASURED_PEAKS copy bandwidth
_L2 = 12.0e12           # B/s
_SECTOR = 32.0

COUNTER_NAMES: Tuple[str, ...] = (
    "DRAM_RT", "DRAM_WT", "L2_RT", "L2_WT", "TEX_RWT", "LOC_O", "SHR_LT", "SHR_WT",
    "INST_F32", "INST_F64", "INST_INT", "INST_MISC", "INST_LDST", "INST_CONT", "INST_BCONV",
    "INST_EXE", "INST_ISSUE_U", "DRAM_U", "L2_U", "TEX_U", "SHR_U", "SM_E", "WARP_E",
    "WARP_NP_E",
)


def _enumerate(params: Sequence[Tuple[str, Sequence[float]]],
               valid: Callable[[Dict[str, np.ndarray]], np.ndarray], target: int,
               seed: int) -> Tuple[List[TuningParameter], np.ndarray]:
    tps = [TuningParameter.make(name, vals) for name, vals in params]
    grid = np.array(list(itertools.product(*(p.values for p in tps))), dtype=np.float64)
    cols = {p.name: grid[:, j] for j, p in enumerate(tps)}
    keep = valid(cols)
    grid = grid[keep]
    if grid.shape[0] < target:
        raise ValueError(f"constraint set leaves {grid.shape[0]} < {target} configurations")
    if grid.shape[0] > target:
        pick = np.sort(np.random.default_rng(seed).permutation(grid.shape[0])[:target])
        grid = grid[pick]
    return tps, np.ascontiguousarray(grid)


def _model(n, *, flops, fp32_inst, int_inst, ldst_inst, ctrl_inst, bconv_inst, misc_inst,
           dram_rd, dram_wr, l2_rd, l2_wr, tex_req, shr_ld, shr_st, local_st, threads,
           block_threads, occupancy, warp_eff, pred_eff, pipe_rate, pipe_eff=1.0,
           mem_eff=1.0):
    """Counters + runtime of one launch per configuration (all arrays of n)."""
    warps_inst = (fp32_inst + int_inst + ldst_inst + ctrl_inst + bconv_inst + misc_inst) / (
        32.0 * warp_eff * pred_eff)
    blocks = np.ceil(threads / block_threads)
    sm_fill = np.minimum(1.0, blocks / B200_SMS)
    waves = np.ceil(blocks / (B200_SMS * np.maximum(1.0, occupancy)))
    tail = blocks / (waves * B200_SMS * np.maximum(1.0, occupancy))
    lat_hide = np.clip(occupancy / 8.0, 0.15, 1.0) * sm_fill * np.clip(tail, 0.3, 1.0)
    t_dram = (dram_rd + dram_wr) * _SECTOR / (_HBM * lat_hide * mem_eff)
    t_l2 = (l2_rd + l2_wr) * _SECTOR / (_L2 * lat_hide)
    t_tex = tex_req / (B200_SMS * _CLOCK * 0.5 * lat_hide)
    t_shr = (shr_ld + shr_st) / (B200_SMS * _CLOCK * lat_hide)
    t_issue = warps_inst / (B200_SMS * 4 * _CLOCK * np.clip(occupancy / 4.0, 0.25, 1.0) * sm_fill)
    t_fp = flops / (B200_SMS * pipe_rate * _CLOCK * sm_fill * pipe_eff)
    t_local = local_st * _SECTOR / (_L2 * 0.5)
    busy = np.maximum.reduce([t_dram, t_l2, t_tex, t_shr, t_issue, t_fp, t_local])
    # overlap is imperfect: add a fraction of the second-largest term
    stack = np.sort(np.stack([t_dram, t_l2, t_tex, t_shr, t_issue, t_fp, t_local]), axis=0)
    runtime_s = busy + 0.6 * stack[-2] + 0.3 * stack[-3] + 2.5e-6
    # run-to-run jitter (+-3%), a fixed function of the configuration row so
    # that plateaus of equal model time break up as real measurements do
    jitter = np.sin(np.arange(n) * 12.9898 + 78.233) * 43758.5453
    runtime_s = runtime_s * (1.0 + 0.03 * (2.0 * (jitter - np.floor(jitter)) - 1.0))
    c = {
        "DRAM_RT": dram_rd, "DRAM_WT": dram_wr, "L2_RT": l2_rd, "L2_WT": l2_wr,
        "TEX_RWT": tex_req, "LOC_O": local_st, "SHR_LT": shr_ld, "SHR_WT": shr_st,
        "INST_F32": fp32_inst, "INST_F64": np.zeros(n), "INST_INT": int_inst,
        "INST_MISC": misc_inst, "INST_LDST": ldst_inst, "INST_CONT": ctrl_inst,
        "INST_BCONV": bconv_inst, "INST_EXE": warps_inst,
        "INST_ISSUE_U": np.clip(100.0 * t_issue / runtime_s, 0.0, 100.0),
        "DRAM_U": np.clip(10.0 * t_dram / runtime_s, 0.0, 10.0),
        "L2_U": np.clip(100.0 * t_l2 / runtime_s, 0.0, 100.0),
        "TEX_U": np.clip(10.0 * t_tex / runtime_s, 0.0, 10.0),
        "SHR_U": np.clip(10.0 * t_shr / runtime_s, 0.0, 10.0),
        "SM_E": np.clip(100.0 * sm_fill * np.clip(tail, 0.5, 1.0), 0.0, 100.0),
        "WARP_E": np.clip(100.0 * warp_eff, 0.0, 100.0),
        "WARP_NP_E": np.clip(100.0 * pred_eff, 0.0, 100.0),
    }
    for k in c:
        c[k] = np.round(np.broadcast_to(np.asarray(c[k], dtype=np.float64), (n,)).copy(), 6)
    runtime_us = np.round(runtime_s * 1e6, 4)
    return runtime_us, c


def _dataset(name, tps, grid, runtime_us, counters, threads) -> Dataset:
    space = TuningSpace.from_assignments(tps, grid)
    cm = np.stack([counters[k] for k in COUNTER_NAMES], axis=1)
    return Dataset(space, B200_ARCH, name, runtime_us=runtime_us,
                   global_threads=np.maximum(1, np.round(threads)).astype(np.int64),
                   counter_names=COUNTER_NAMES, counter_matrix=cm)


def _transpose_valid(p):
    tx = p["TILE"] / p["VEC"]
    threads = tx * p["BLOCK_Y"]
    return ((p["BLOCK_Y"] <= p["TILE"]) & (threads >= 32) & (threads <= 1024)
            & (tx >= 2) & ((p["USE_SMEM"] == 1) | (p["PAD"] == 0)))


TRANSPOSE_PARAMS = [("TILE", [8, 16, 32, 64]), ("VEC", [1, 2, 4]), ("PAD", [0, 1]),
                    ("BLOCK_Y", [1, 2, 4, 8, 16, 32]), ("USE_SMEM", [0, 1]), ("DIAG", [0, 1]),
                    ("UNROLL", [1, 2, 4, 8]), ("WORK_X", [1, 2])]


def transpose(size: int = 8192, target: int = 1784) -> Dataset:
    tps, g = _enumerate(TRANSPOSE_PARAMS, _transpose_valid, target, seed=1784)
    T, V, PAD, BY, SM, DG, UN, WX = (g[:, j] for j in range(8))
    n = g.shape[0]
    elems = float(size) * size
    sectors = elems * 4.0 / _SECTOR
    tx = T / V
    block_threads = tx * BY
    threads = elems / (V * (T / BY) * WX) / 1.0
    # without shared memory the writes are strided: a warp touches 32 sectors
    wr_amp = np.where(SM == 1, 1.0, np.minimum(8.0, 8.0 / V))
    rd_amp = 1.0 + 0.04 * (T == 8) + 0.02 * (DG == 0) * (T >= 32)
    dram_rd = sectors * rd_amp * (1.0 + 0.03 * (DG == 0))
    dram_wr = sectors * (1.0 + 0.35 * (wr_amp - 1.0) / 7.0 + 0.02 * (DG == 0))
    l2_rd = sectors * rd_amp
    l2_wr = sectors * wr_amp
    conflicts = np.where(PAD == 1, 1.0, np.where(T >= 32, 32.0 / V, T / (2.0 * V)))
    shr_st = np.where(SM == 1, elems / (32.0 * V) * V, 0.0)
    shr_ld = np.where(SM == 1, elems / (32.0 * V) * np.maximum(1.0, conflicts), 0.0)
    per_thread_elems = elems / threads
    ldst = elems / V * np.where(SM == 1, 2.0, 1.0) * 2.0 / 2.0 + elems / V
    intops = elems * (2.5 + 1.5 / V) * (1.0 + 0.3 / UN) + threads * 6
    ctrl = threads * per_thread_elems / (V * UN) + threads * 2
    bconv = threads * 1.0
    misc = np.where(SM == 1, threads * per_thread_elems / (T * V) * 2.0 + threads, threads)
    occ = np.clip(2048.0 / block_threads, 1, 32) * np.where(
        SM == 1, np.clip(200e3 / (T * (T + PAD) * 4.0 * 2), 0.25, 1.0), 1.0)
    occ = np.minimum(occ, 32.0)
    warp_eff = np.clip(np.minimum(1.0, block_threads / 32.0), 0.05, 1.0)
    pred_eff = np.full(n, 0.985)
    # bytes in flight per thread and partition camping set the HBM efficiency
    mem_eff = np.clip(0.45 + 0.09 * np.log2(V * UN * WX) + 0.04 * np.log2(T / 8.0), 0.3, 1.0)
    mem_eff *= np.where((DG == 0) & (T >= 32), 0.93, 1.0) * np.where(BY >= 16, 0.95, 1.0)
    runtime, c = _model(n, flops=np.zeros(n), fp32_inst=np.zeros(n) + elems * 0.0,
                        int_inst=intops, ldst_inst=ldst, ctrl_inst=ctrl, bconv_inst=bconv,
                        misc_inst=misc, dram_rd=dram_rd, dram_wr=dram_wr, l2_rd=l2_rd,
                        l2_wr=l2_wr, tex_req=elems / (32.0 * V), shr_ld=shr_ld, shr_st=shr_st,
                        local_st=np.zeros(n), threads=threads, block_threads=block_threads,
                        occupancy=occ, warp_eff=warp_eff, pred_eff=pred_eff,
                        pipe_rate=128.0, mem_eff=mem_eff)
    return _dataset("transpose-8192", tps, g, runtime, c, threads)


GEMM_PARAMS = [("MWG", [16, 32, 64, 128]), ("NWG", [16, 32, 64, 128]), ("KWG", [16, 32]),
               ("MDIMC", [8, 16, 32]), ("NDIMC", [8, 16, 32]), ("VWM", [1, 2, 4, 8]),
               ("VWN", [1, 2, 4, 8]), ("SA", [0, 1]), ("SB", [0, 1]), ("TC", [0, 1])]
GEMM_FULL_PARAMS = [("MWG", [16, 32, 64, 128]), ("NWG", [16, 32, 64, 128]), ("KWG", [16, 32]),
                    ("MDIMC", [8, 16, 32]), ("NDIMC", [8, 16, 32]), ("MDIMA", [8, 16, 32]),
                    ("NDIMB", [8, 16, 32]), ("KWI", [2, 8]), ("VWM", [1, 2, 4, 8]),
                    ("VWN", [1, 2, 4, 8]), ("STRM", [0, 1]), ("STRN", [0, 1]), ("SA", [0, 1]),
                    ("SB", [0, 1])]


def _gemm_valid(p, full=False):
    ok = ((p["MWG"] % (p["MDIMC"] * p["VWM"]) == 0) & (p["NWG"] % (p["NDIMC"] * p["VWN"]) == 0)
          & (p["MDIMC"] * p["NDIMC"] >= 64) & (p["MDIMC"] * p["NDIMC"] <= 1024))
    if full:
        ok &= ((p["MWG"] % (p["MDIMA"] * p["VWM"]) == 0)
               & (p["NWG"] % (p["NDIMB"] * p["VWN"]) == 0)
               & ((p["MDIMC"] * p["NDIMC"]) % p["MDIMA"] == 0)
               & ((p["MDIMC"] * p["NDIMC"]) % p["NDIMB"] == 0))
    else:
        ok &= (p["TC"] == 0) | ((p["SA"] == 1) & (p["SB"] == 1))
    return ok


def gemm(m: int = 2048, target: int = 5788, full: bool = False) -> Dataset:
    if full:
        target = 205216
    tps, g = _enumerate(GEMM_FULL_PARAMS if full else GEMM_PARAMS,
                        lambda p: _gemm_valid(p, full), target,
                        seed=5788 if not full else 205216)
    col = {p.name: g[:, j] for j, p in enumerate(tps)}
    n = g.shape[0]
    MWG, NWG, KWG = col["MWG"], col["NWG"], col["KWG"]
    MD, ND, VWM, VWN = col["MDIMC"], col["NDIMC"], col["VWM"], col["VWN"]
    SA, SB = col["SA"], col["SB"]
    TC = col.get("TC", np.zeros(n))
    block_threads = MD * ND
    blocks = (m / MWG) * (m / NWG)
    threads = blocks * block_threads
    flops = 2.0 * m * m * m
    reuse_a = np.where(SA == 1, NWG, ND * VWN * 0.5 + 1)
    reuse_b = np.where(SB == 1, MWG, MD * VWM * 0.5 + 1)
    gbytes_rd = 4.0 * m * m * m * (1.0 / reuse_a + 1.0 / reuse_b)
    l2_rd = gbytes_rd / _SECTOR
    dram_rd = l2_rd * np.clip(0.6 * (m * m * 8.0 / 126e6) + 0.05, 0.05, 1.0) + 2 * m * m * 4 / _SECTOR
    dram_wr = np.full(n, m * m * 4.0 / _SECTOR)
    l2_wr = dram_wr.copy()
    shr_st = (SA * m * m * m / NWG + SB * m * m * m / MWG) / (32.0 * np.minimum(VWM, 4))
    shr_ld = (SA * m * m * m / (ND * VWN) + SB * m * m * m / (MD * VWM)) / 32.0 * 2.0
    regs_tile = (MWG / MD) * (NWG / ND)
    spill = np.where(regs_tile > 128, (regs_tile - 128) * threads * 4.0, 0.0)
    fp32 = np.where(TC == 1, flops / 64.0, flops / 2.0)
    ldst = (shr_ld + shr_st) * 32.0 + gbytes_rd / (4.0 * np.maximum(VWM, VWN))
    intops = fp32 * 0.08 + threads * 40
    ctrl = m * m * m / (KWG * regs_tile) * 2.0 / 32.0 * 32.0
    bconv = np.where(TC == 1, flops / 256.0, threads * 2.0)
    misc = threads * 4.0 + (SA + SB) * m * m * m / (KWG * 64.0)
    smem_b = 4.0 * KWG * (SA * MWG + SB * NWG)
    occ = np.minimum(2048.0 / block_threads, np.minimum(228e3 / np.maximum(smem_b, 1.0), 32.0))
    occ = np.minimum(occ, np.maximum(1.0, 65536.0 / (block_threads * np.minimum(255.0, regs_tile + 32))))
    warp_eff = np.full(n, 1.0)
    pred_eff = np.full(n, 0.995)
    pipe = np.where(TC == 1, 1024.0, 128.0)
    # FMA-pipe efficiency grows with the register tile (ILP) and vector width
    pipe_eff = np.clip(regs_tile / 32.0, 0.15, 1.0) * (0.8 + 0.05 * np.minimum(VWM, 4.0))
    pipe_eff *= np.where(regs_tile > 128, 0.6, 1.0)
    runtime, c = _model(n, flops=flops, fp32_inst=fp32, int_inst=intops, ldst_inst=ldst,
                        ctrl_inst=ctrl, bconv_inst=bconv, misc_inst=misc, dram_rd=dram_rd,
                        dram_wr=dram_wr, l2_rd=l2_rd, l2_wr=l2_wr,
                        tex_req=gbytes_rd / (128.0 * np.maximum(VWM, VWN)), shr_ld=shr_ld,
                        shr_st=shr_st, local_st=spill / _SECTOR, threads=threads,
                        block_threads=block_threads, occupancy=occ, warp_eff=warp_eff,
                        pred_eff=pred_eff, pipe_rate=pipe, pipe_eff=pipe_eff)
    return _dataset("gemm-full-2048" if full else "gemm-2048", tps, g, runtime, c, threads)


def gemm_full() -> Dataset:
    return gemm(full=True)


def _pairwise(name, label, target, seed, n_bodies, params, valid, per_pair_flops, inner_mufu):
    tps, g = _enumerate(params, valid, target, seed)
    col = {p.name: g[:, j] for j, p in enumerate(tps)}
    n = g.shape[0]
    BS = col["BLOCK"]
    OUT = col.get("OUTER", np.ones(n))
    UN = col.get("UNROLL", np.ones(n))
    SMEM = col.get("USE_SMEM", np.ones(n))
    VEC = col.get("VEC", np.ones(n))
    RSQ = col.get("FAST_RSQRT", np.zeros(n))
    threads = np.ceil(n_bodies / OUT)
    pairs = float(n_bodies) * n_bodies
    fp32 = pairs * per_pair_flops * np.where(RSQ == 1, 0.9, 1.0)
    misc = pairs * inner_mufu * np.where(RSQ == 1, 0.35, 1.0)
    ldst = pairs / OUT * np.where(SMEM == 1, 1.0 / VEC, 1.0 / VEC) + threads * 8
    shr_ld = np.where(SMEM == 1, pairs / (OUT * 32.0 * VEC), 0.0)
    shr_st = np.where(SMEM == 1, n_bodies * threads / BS / 32.0, 0.0)
    tex = np.where(SMEM == 1, n_bodies * threads / BS / 32.0, pairs / (OUT * 32.0))
    l2_rd = tex * 4.0
    dram_rd = np.full(n, n_bodies * 16.0 / _SECTOR) * (1.0 + 0.1 * (SMEM == 0))
    dram_wr = np.full(n, n_bodies * 12.0 / _SECTOR)
    ctrl = pairs / (OUT * UN * 32.0) * 32.0
    intops = pairs / (OUT * UN) * 2.0 + threads * 20
    occ = np.minimum(2048.0 / BS, 32.0) * np.where(OUT >= 8, 0.5, 1.0)
    warp_eff = np.clip(threads / (np.ceil(threads / BS) * BS), 0.1, 1.0)
    runtime, c = _model(n, flops=fp32, fp32_inst=fp32, int_inst=intops, ldst_inst=ldst,
                        ctrl_inst=ctrl, bconv_inst=threads * 4.0, misc_inst=misc,
                        dram_rd=dram_rd, dram_wr=dram_wr, l2_rd=l2_rd, l2_wr=dram_wr,
                        tex_req=tex, shr_ld=shr_ld, shr_st=shr_st, local_st=np.zeros(n),
                        threads=threads, block_threads=BS, occupancy=occ, warp_eff=warp_eff,
                        pred_eff=np.full(n, 0.99), pipe_rate=128.0,
                        pipe_eff=np.clip(0.4 + 0.1 * np.log2(OUT) + 0.04 * np.log2(UN)
                                         + 0.05 * (SMEM == 1) - 0.12 * (OUT >= 16), 0.2, 1.0))
    return _dataset(label, tps, g, runtime, c, threads)


NBODY_PARAMS = [("BLOCK", [32, 64, 128, 256, 512, 1024]), ("OUTER", [1, 2, 4, 8, 16]),
                ("UNROLL", [1, 2, 4, 8, 16, 32]), ("USE_SMEM", [0, 1]), ("VEC", [1, 2, 4]),
                ("FAST_RSQRT", [0, 1]), ("SOA", [0, 1])]


def _nbody_valid(p):
    return (p["UNROLL"] <= p["BLOCK"]) & ((p["USE_SMEM"] == 1) | (p["VEC"] <= 2))


def nbody(bodies: int = 16384, target: int = 3134) -> Dataset:
    return _pairwise("nbody", f"nbody-{bodies}", target, 3134, bodies, NBODY_PARAMS,
                     _nbody_valid, 20.0, 1.0)


COULOMB_PARAMS = [("BLOCK", [32, 64, 128, 256]), ("Z_ITERATIONS", [1, 2, 4, 8, 16, 32]),
                  ("INNER_UNROLL", [0, 1, 2, 4, 8]), ("USE_SMEM", [0, 1]), ("USE_SOA", [0, 1]),
                  ("VECTOR_TYPE", [1, 2, 4]), ("USE_CONST", [0])]


def _coulomb_valid(p):
    return (((p["USE_SMEM"] == 0) | (p["USE_CONST"] == 0))
            & ((p["VECTOR_TYPE"] == 1) | (p["USE_SOA"] == 1))
            & (p["INNER_UNROLL"] <= p["Z_ITERATIONS"] * 2))


def coulomb(grid: int = 256, atoms: int = 256, target: int = 210) -> Dataset:
    tps, g = _enumerate(COULOMB_PARAMS, _coulomb_valid, target, seed=210)
    col = {p.name: g[:, j] for j, p in enumerate(tps)}
    n = g.shape[0]
    BS, Z = col["BLOCK"], col["Z_ITERATIONS"]
    UN, SM, SOA, VT = col["INNER_UNROLL"], col["USE_SMEM"], col["USE_SOA"], col["VECTOR_TYPE"]
    points = float(grid) ** 3
    inter = points * atoms
    threads = points / Z
    fp32 = inter * (9.0 - 0.5 * (Z > 1))
    misc = inter * 1.0
    ldst = inter / Z * np.where(SM == 1, 1.0, 1.0) / VT * np.where(SOA == 1, 1.0, 4.0)
    shr_ld = np.where(SM == 1, inter / (Z * 32.0 * VT), 0.0)
    shr_st = np.where(SM == 1, atoms * threads / BS / 32.0, 0.0)
    tex = np.where(SM == 1, atoms * threads / BS / 32.0, inter / (Z * 32.0 * VT))
    dram_wr = np.full(n, points * 4.0 / _SECTOR)
    dram_rd = np.full(n, atoms * 16.0 / _SECTOR) + dram_wr * 0.05
    ctrl = inter / (Z * np.maximum(UN, 1)) / 8.0
    intops = inter / Z * 1.5 + threads * 30
    occ = np.minimum(2048.0 / BS, 32.0) * np.where(Z >= 16, 0.5, 1.0)
    # ILP from the z-coarsening and unrolling, vector loads of atom data
    pipe_eff = np.clip(0.35 + 0.1 * np.log2(Z) + 0.04 * np.log2(1.0 + UN) + 0.04 * (VT - 1.0)
                       - 0.05 * (SM == 0) * (BS >= 128), 0.2, 1.0)
    pipe_eff *= np.where(Z >= 32, 0.8, 1.0)
    runtime, c = _model(n, flops=fp32, fp32_inst=fp32, int_inst=intops, ldst_inst=ldst,
                        ctrl_inst=ctrl, bconv_inst=threads * 3.0, misc_inst=misc,
                        dram_rd=dram_rd, dram_wr=dram_wr, l2_rd=tex * 4.0 + dram_rd,
                        l2_wr=dram_wr, tex_req=tex, shr_ld=shr_ld, shr_st=shr_st,
                        local_st=np.zeros(n), threads=threads, block_threads=BS,
                        occupancy=occ, warp_eff=np.full(n, 1.0), pred_eff=np.full(n, 0.995),
                        pipe_rate=128.0, pipe_eff=pipe_eff)
    return _dataset(f"coulomb-{grid}^3x{atoms}", tps, g, runtime, c, threads)


CONV_PARAMS = [("TBX", [8, 16, 32, 64]), ("TBY", [1, 2, 4, 8, 16]), ("WPTX", [1, 2, 4, 8]),
               ("WPTY", [1, 2, 4, 8]), ("VW", [1, 2, 4]), ("LOCAL", [0, 1, 2]),
               ("PAD", [0, 1]), ("UNROLL_F", [0, 1]), ("CACHE_F", [0, 1]), ("REVERSE", [0, 1])]


def _conv_valid(p):
    t = p["TBX"] * p["TBY"]
    return ((t >= 32) & (t <= 1024) & (p["WPTX"] % p["VW"] == 0)
            & ((p["LOCAL"] > 0) | (p["PAD"] == 0)) & (p["WPTX"] * p["WPTY"] <= 32))


def conv(size: int = 4096, filt: int = 7, target: int = 3928) -> Dataset:
    tps, g = _enumerate(CONV_PARAMS, _conv_valid, target, seed=3928)
    col = {p.name: g[:, j] for j, p in enumerate(tps)}
    n = g.shape[0]
    TBX, TBY, WX, WY, VW = col["TBX"], col["TBY"], col["WPTX"], col["WPTY"], col["VW"]
    LOC, PAD, UF, CF = col["LOCAL"], col["PAD"], col["UNROLL_F"], col["CACHE_F"]
    px = float(size) * size
    taps = filt * filt
    threads = px / (WX * WY)
    block_threads = TBX * TBY
    fp32 = px * taps * 2.0 / 2.0
    tile_w, tile_h = TBX * WX + filt - 1, TBY * WY + filt - 1
    halo = (tile_w * tile_h) / (TBX * WX * TBY * WY)
    gread = np.where(LOC > 0, px * halo, px * taps / np.maximum(1.0, WX * WY * 0.5))
    l2_rd = gread * 4.0 / _SECTOR
    dram_rd = px * 4.0 / _SECTOR * (1.0 + 0.1 * (LOC == 0))
    dram_wr = np.full(n, px * 4.0 / _SECTOR)
    conflicts = np.where(PAD == 1, 1.0, np.where(LOC == 2, 2.0, 4.0))
    shr_ld = np.where(LOC > 0, px * taps / (32.0 * VW) * conflicts / np.where(LOC == 2, 2.0, 1.0), 0.0)
    shr_st = np.where(LOC > 0, px * halo / 32.0, 0.0)
    ldst = shr_ld * 32.0 + gread / VW
    ctrl = px * taps / np.where(UF == 1, taps, 1.0) / 32.0 * 32.0 / 8.0
    intops = px * taps * np.where(UF == 1, 0.3, 1.2) + threads * 20
    misc = threads * np.where(CF == 1, 6.0, 2.0) + px * taps * (CF == 0) * 0.05
    smem_b = 4.0 * tile_w * (tile_h + PAD)
    occ = np.minimum(2048.0 / block_threads, np.where(LOC > 0, 228e3 / smem_b, 32.0))
    occ = np.clip(occ, 1.0, 32.0)
    warp_eff = np.clip(np.minimum(1.0, block_threads / 32.0), 0.1, 1.0)
    runtime, c = _model(n, flops=fp32, fp32_inst=fp32, int_inst=intops, ldst_inst=ldst,
                        ctrl_inst=ctrl, bconv_inst=threads * 2.0, misc_inst=misc,
                        dram_rd=dram_rd, dram_wr=dram_wr, l2_rd=l2_rd, l2_wr=dram_wr,
                        tex_req=gread / (32.0 * VW), shr_ld=shr_ld, shr_st=shr_st,
                        local_st=np.zeros(n), threads=threads, block_threads=block_threads,
                        occupancy=occ, warp_eff=warp_eff, pred_eff=np.full(n, 0.98),
                        pipe_rate=128.0,
                        pipe_eff=np.clip(0.3 + 0.08 * np.log2(WX * WY) + 0.1 * UF + 0.05 * CF
                                         + 0.03 * np.log2(VW), 0.2, 1.0))
    return _dataset(f"conv-{size}-{filt}x{filt}", tps, g, runtime, c, threads)


# (parameters, constraint, Table-2 size, subsample seed) of every space: the
# live benchmarks (live.py) enumerate exactly the same configurations
SPACE_SPECS = {
    "coulomb": (COULOMB_PARAMS, _coulomb_valid, 210, 210),
    "transpose": (TRANSPOSE_PARAMS, _transpose_valid, 1784, 1784),
    "nbody": (NBODY_PARAMS, _nbody_valid, 3134, 3134),
    "conv": (CONV_PARAMS, _conv_valid, 3928, 3928),
    "gemm": (GEMM_PARAMS, _gemm_valid, 5788, 5788),
    "gemm_full": (GEMM_FULL_PARAMS, lambda p: _gemm_valid(p, True), 205216, 205216),
}


def space_of(name: str) -> TuningSpace:
    """The tuning space of a benchmark (same configurations, same order as
    the synthetic dataset of that name)."""
    params, valid, target, seed = SPACE_SPECS[name]
    tps, g = _enumerate(params, valid, target, seed)
    return TuningSpace.from_assignments(tps, g)


SPACES = {
    "coulomb": coulomb,
    "transpose": transpose,
    "nbody": nbody,
    "conv": conv,
    "gemm": gemm,
    "gemm_full": gemm_full,
}


def stress(n: int = 1 << 20, seed: int = 1) -> Dataset:
    """The scoring microbenchmark's inputs (SURVEY
    section 8d) as a replay dataset: every operation counter (the exact
    model's table columns) uniform(1, 1e6) with 2% exact zeros, utilisations
    uniform over their ranges, runtimes uniform(100, 1000) us.  The space is
    the first n points of a 6-parameter grid of 16 values each.  At n >= 1M
    the 19-column table (152 MB at 1M, 608 MB at 4M) no longer fits the
    126 MB L2, so the search kernel's table reads come from HBM."""
    if not 1 <= n <= 16 ** 6:
        raise ValueError("stress spaces hold 1 .. 16^6 configurations")
    rng = np.random.default_rng(seed)
    idx = np.arange(n, dtype=np.int64)
    grid = np.stack([(idx >> (4 * k)) & 15 for k in range(6)], axis=1).astype(np.float64)
    tps = [TuningParameter(name=f"P{k}", values=tuple(float(v) for v in range(16)),
                           is_binary=False) for k in range(6)]
    cm = np.empty((n, len(COUNTER_NAMES)))
    for j, name in enumerate(COUNTER_NAMES):
        if name in ("DRAM_U", "TEX_U", "SHR_U"):
            col = rng.uniform(0.0, 10.0, n)
        elif name in ("L2_U", "SM_E", "WARP_E", "WARP_NP_E", "INST_ISSUE_U"):
            col = rng.uniform(0.0, 100.0, n)
        else:
            col = rng.uniform(1.0, 1e6, n)
            col[rng.random(n) < 0.02] = 0.0
        cm[:, j] = col
    threads = rng.integers(1 << 10, 1 << 24, n)
    space = TuningSpace.from_assignments(tps, grid)
    return Dataset(space, B200_ARCH, f"stress-{n}", runtime_us=rng.uniform(100.0, 1000.0, n),
                   global_threads=threads, counter_names=COUNTER_NAMES, counter_matrix=cm)


def required_present(ds: Dataset) -> bool:
    return all(a in ds.counter_names for a in REQUIRED_COUNTERS)

"""Counter vocabulary of the searcher (the reference's counters.py, reduced to
what the hot path and its measurement boundary read).

* ABBREVIATIONS -- canonical catalog order (counters.py:58-105); it is also the
  column order of PredictionTables built from trained model sets
  (models.py:301-304).
* REQUIRED_COUNTERS -- what analyze() reads (bottlenecks.py:21-30), the row
  layout of the device replay counters.
* DELTA_KEYS -- react()'s insertion order (bottlenecks.py:216-229), which is
  the Eq. 16 accumulation order the kernels must follow.
* VOLTA_METRICS -- Volta+ metric names and the factor that brings a reading to
  the canonical pre-Volta scale (Table 1 of the paper); the measurement
  boundary canonicalises raw names with it.
"""

from dataclasses import dataclass, field
from typing import Dict, Tuple

OPS = "ops"
STRESS = "stress"
PRE_VOLTA = "pre_volta"
VOLTA_PLUS = "volta_plus"
GENERATIONS = (PRE_VOLTA, VOLTA_PLUS)
GLOBAL_THREADS = "GLOBAL_THREADS"

_OPS_ORDER = ("DRAM_RT", "DRAM_WT", "L2_RT", "L2_WT", "TEX_RWT", "LOC_O", "SHR_LT", "SHR_WT",
              "INST_F32", "INST_F64", "INST_INT", "INST_MISC", "INST_LDST", "INST_CONT",
              "INST_BCONV", "INST_EXE", "INST_ISSUE_U")
_STRESS_ORDER = ("DRAM_U", "L2_U", "TEX_U", "SHR_U", "SM_E", "WARP_E", "WARP_NP_E")

ABBREVIATIONS: Tuple[str, ...] = _OPS_ORDER + _STRESS_ORDER + (GLOBAL_THREADS,)
KIND: Dict[str, str] = {**{a: OPS for a in _OPS_ORDER}, **{a: STRESS for a in _STRESS_ORDER},
                        GLOBAL_THREADS: OPS}

REQUIRED_COUNTERS: Tuple[str, ...] = (
    "DRAM_RT", "DRAM_WT", "DRAM_U", "L2_RT", "L2_WT", "L2_U", "SHR_LT", "SHR_WT", "SHR_U",
    "TEX_U", "LOC_O", "INST_F32", "INST_F64", "INST_INT", "INST_MISC", "INST_LDST",
    "INST_CONT", "INST_BCONV", "INST_EXE", "INST_ISSUE_U", "WARP_E", "WARP_NP_E", "SM_E",
)

COMPONENT_NAMES: Tuple[str, ...] = (
    "b_dram_read", "b_dram_write", "b_l2_read", "b_l2_write", "b_shared_read",
    "b_shared_write", "b_tex", "b_local", "b_fp32", "b_fp64", "b_int", "b_misc", "b_ldst",
    "b_control", "b_bconv", "b_issue", "b_sm", "b_paral",
)

DELTA_KEYS: Tuple[str, ...] = (
    "DRAM_RT", "DRAM_WT", "L2_RT", "L2_WT", "SHR_LT", "SHR_WT", "TEX_RWT", "LOC_O",
    "INST_F32", "INST_F64", "INST_INT", "INST_MISC", "INST_LDST", "INST_CONT", "INST_BCONV",
    "INST_ISSUE_U", "SM_E", GLOBAL_THREADS,
)

# Volta+ metric name, scale to the canonical (pre-Volta) value range.  All 24
# exist on GB100.
VOLTA_METRICS: Dict[str, Tuple[str, float]] = {
    "DRAM_RT": ("dram__sectors_read.sum", 1.0),
    "DRAM_WT": ("dram__sectors_write.sum", 1.0),
    "L2_RT": ("lts__t_sectors_op_read.sum", 1.0),
    "L2_WT": ("lts__t_sectors_op_write.sum", 1.0),
    "TEX_RWT": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 1.0),
    "LOC_O": ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", 1.0),
    "SHR_LT": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1.0),
    "SHR_WT": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 1.0),
    "INST_F32": ("smsp__sass_thread_inst_executed_op_fp32_pred_on.sum", 1.0),
    "INST_F64": ("smsp__sass_thread_inst_executed_op_fp64_pred_on.sum", 1.0),
    "INST_INT": ("smsp__sass_thread_inst_executed_op_integer_pred_on.sum", 1.0),
    "INST_MISC": ("smsp__sass_thread_inst_executed_op_misc_pred_on.sum", 1.0),
    "INST_LDST": ("smsp__sass_thread_inst_executed_op_memory_pred_on.sum", 1.0),
    "INST_CONT": ("smsp__sass_thread_inst_executed_op_control_pred_on.sum", 1.0),
    "INST_BCONV": ("smsp__sass_thread_inst_executed_op_conversion_pred_on.sum", 1.0),
    "INST_EXE": ("smsp__inst_executed.sum", 1.0),
    "INST_ISSUE_U": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "DRAM_U": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0.1),
    "L2_U": ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1.0),
    "TEX_U": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.avg.pct_of_peak_sustained_active",
              0.1),
    "SHR_U": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
              0.1),
    "SM_E": ("smsp__cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "WARP_E": ("smsp__thread_inst_executed_per_inst_executed.ratio", 100.0 / 32.0),
    "WARP_NP_E": ("smsp__thread_inst_executed_per_inst_executed.pct", 1.0),
}
_BY_VOLTA = {name: (abbr, scale) for abbr, (name, scale) in VOLTA_METRICS.items()}

# Pre-Volta (nvprof event/metric) names; readings are canonical as they come.
PRE_VOLTA_NAMES: Dict[str, str] = {
    "DRAM_RT": "dram_read_transactions", "DRAM_WT": "dram_write_transactions",
    "L2_RT": "l2_read_transactions", "L2_WT": "l2_write_transactions",
    "TEX_RWT": "tex_cache_transactions", "LOC_O": "local_memory_overhead",
    "SHR_LT": "shared_load_transactions", "SHR_WT": "shared_store_transactions",
    "INST_F32": "inst_fp_32", "INST_F64": "inst_fp_64", "INST_INT": "inst_integer",
    "INST_MISC": "inst_misc", "INST_LDST": "inst_compute_ld_st", "INST_CONT": "inst_control",
    "INST_BCONV": "inst_bit_convert", "INST_EXE": "inst_executed",
    "INST_ISSUE_U": "issue_slot_utilization", "DRAM_U": "dram_utilization",
    "L2_U": "l2_utilization", "TEX_U": "tex_utilization", "SHR_U": "shared_utilization",
    "SM_E": "sm_efficiency", "WARP_E": "warp_execution_efficiency",
    "WARP_NP_E": "warp_nonpred_execution_efficiency",
}
_BY_PRE_VOLTA = {name: abbr for abbr, name in PRE_VOLTA_NAMES.items()}


@dataclass(frozen=True)
class ArchProfile:
    """Identity and counter dialect of one GPU (counters.py:140-158)."""

    name: str
    generation: str
    cores: int
    overrides: Dict[str, Tuple[str, float]] = field(default_factory=dict)

    def __post_init__(self):
        if self.generation not in GENERATIONS:
            raise ValueError(f"generation must be one of {GENERATIONS}, got {self.generation!r}")
        if self.cores < 1:
            raise ValueError(f"cores must be >= 1, got {self.cores}")


def generation_code(arch) -> int:
    """0 pre_volta / 1 volta_plus, the device encoding."""
    return 0 if arch.generation == PRE_VOLTA else 1


def canonicalize(raw_name: str, value: float, arch) -> Tuple[str, float]:
    """Raw counter reading -> (abbreviation, canonical value) (counters.py:161-180).

    Order: arch overrides, then the generation's catalog names, then the
    canonical abbreviations verbatim.
    """
    overrides = getattr(arch, "overrides", {}) or {}
    if raw_name in overrides:
        abbr, scale = overrides[raw_name]
        if abbr not in KIND:
            raise KeyError(f"arch override for {raw_name!r} targets unknown counter {abbr!r}")
        return abbr, value * scale
    if arch.generation == VOLTA_PLUS and raw_name in _BY_VOLTA:
        abbr, scale = _BY_VOLTA[raw_name]
        return abbr, value * scale
    if arch.generation == PRE_VOLTA and raw_name in _BY_PRE_VOLTA:
        return _BY_PRE_VOLTA[raw_name], value
    if raw_name in KIND:
        return raw_name, value
    raise KeyError(f"counter name {raw_name!r} is not known for generation {arch.generation}")


def dataset_counter_names(dataset) -> Tuple[str, ...]:
    """Counters present in a dataset, catalog order (space.py:163-167)."""
    names = getattr(dataset, "counter_names", None)
    if names is not None:
        return tuple(names)
    present = set(dataset.records[0].counters)
    return tuple(a for a in ABBREVIATIONS if a in present)


def modeled_counters(dataset) -> Tuple[str, ...]:
    """OPS counters present, then GLOBAL_THREADS, then SM_E (models.py:344-351)."""
    present = set(dataset_counter_names(dataset))
    names = [a for a in _OPS_ORDER if a in present]
    names.append(GLOBAL_THREADS)
    if "SM_E" in present:
        names.append("SM_E")
    return tuple(names)

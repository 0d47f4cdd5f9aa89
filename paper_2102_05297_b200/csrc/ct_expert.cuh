// ct_expert.cuh -- the expert system (Eqs. 6-15), host+device.
//
// analyze() follows bottlenecks.py:115-195 and react() bottlenecks.py:202-230
// operation for operation, so every component is bit-identical to the
// reference's Python float arithmetic.  Counter inputs arrive in
// REQUIRED_COUNTERS order (bottlenecks.py:21-30); the 18 bottleneck
// components and the 18 delta keys share one index (COMPONENT_NAMES order,
// bottlenecks.py:54-55 == react() insertion order).
#pragma once
#include "ct_hd.cuh"

namespace ct {

enum Req {
    DRAM_RT, DRAM_WT, DRAM_U, L2_RT, L2_WT, L2_U, SHR_LT, SHR_WT, SHR_U, TEX_U, LOC_O,
    INST_F32, INST_F64, INST_INT, INST_MISC, INST_LDST, INST_CONT, INST_BCONV,
    INST_EXE, INST_ISSUE_U, WARP_E, WARP_NP_E, SM_E_, N_REQ
};

// component / delta-key index
enum Comp {
    B_DRAM_READ, B_DRAM_WRITE, B_L2_READ, B_L2_WRITE, B_SHARED_READ, B_SHARED_WRITE,
    B_TEX, B_LOCAL,
    B_FP32, B_FP64, B_INT, B_MISC, B_LDST, B_CONTROL, B_BCONV, B_ISSUE,
    B_SM, B_PARAL, N_COMP
};

CT_HD double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }
CT_HD double clamp_signed(double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); }
// _traffic_share (bottlenecks.py:109-112)
CT_HD double share(double part, double total) { return total > 0.0 ? dvd(part, total) : 0.0; }
// Python max()/min() keep the first of equal arguments
CT_HD double pymax(double a, double b) { return b > a ? b : a; }

CT_HD bool degenerate_of(const double* c) {
    return c[INST_EXE] <= 0.0 || c[WARP_E] <= 0.0 || c[WARP_NP_E] <= 0.0;
}

// Component k of analyze() (COMPONENT_NAMES index), clamped.  One function
// per component lets one warp evaluate the 18 components on 18 lanes while
// analyze() below, the scalar form, calls the very same code.
CT_HD double analyze_component(const double* c, int k, int generation, int64_t cores,
                               int64_t global_threads, bool degenerate) {
    double v;
    if (k < B_TEX) {                                  // memory read/write pairs
        const int rd = (k < 2) ? DRAM_RT : (k < 4 ? L2_RT : SHR_LT);
        const int util = (k < 2) ? DRAM_U : (k < 4 ? L2_U : SHR_U);
        const double tot = add(c[rd], c[rd + 1]);
        v = dvd(mul(share(c[rd + (k & 1)], tot), c[util]), 10.0);
    } else if (k == B_TEX) {
        v = dvd(c[TEX_U], 10.0);
    } else if (k == B_LOCAL) {
        const double busiest = pymax(pymax(c[DRAM_U], c[L2_U]), c[TEX_U]);
        v = dvd(mul(dvd(c[LOC_O], 100.0), busiest), 10.0);
    } else if (k <= B_ISSUE) {                        // instruction classes
        if (degenerate) return 0.0;
        const double fitted = mul(mul(mul(32.0, c[INST_EXE]), dvd(100.0, c[WARP_E])),
                                  dvd(100.0, c[WARP_NP_E]));
        if (k < B_ISSUE) {
            double util;
            if (generation == 0) {
                util = dvd(c[INST_ISSUE_U], 100.0);
            } else {
                const double u = dvd(c[INST_ISSUE_U], 50.0);
                util = (u < 1.0) ? u : 1.0;           // min(1.0, u)
            }
            v = mul(dvd(c[INST_F32 + (k - B_FP32)], fitted), util);
        } else {
            double util_max = dvd(c[INST_F32], fitted);
            for (int j = 1; j < 7; ++j) util_max = pymax(util_max, dvd(c[INST_F32 + j], fitted));
            v = dvd(mul(util_max, sub(100.0, c[INST_ISSUE_U])), 100.0);
        }
    } else if (k == B_SM) {
        v = dvd(sub(100.0, c[SM_E_]), 100.0);
    } else {
        const double sat = (double)(cores * 5);
        const double par = dvd(sub(sat, (double)global_threads), sat);
        v = par > 0.0 ? par : 0.0;                    // max(0.0, par)
    }
    return clamp01(v);
}

#if defined(__CUDACC__)
// Warp form (lane k evaluates component k, all 32 lanes call it converged):
// the same operations as analyze_component, but the b_issue lane takes the
// seven per-class ratios dvd(c[INST_F32 + j], fitted) from lanes 8..14,
// which compute exactly those values for their own components, instead of
// redoing seven dependent divisions.  Bit-identical to analyze_component.
__device__ __forceinline__ double analyze_component_warp(const double* c, int k, int generation,
                                                         int64_t cores, int64_t global_threads,
                                                         bool degenerate) {
    const bool inst = (k >= B_FP32) && (k <= B_ISSUE) && !degenerate;
    double ratio = 0.0;
    if (inst) {
        const double fitted = mul(mul(mul(32.0, c[INST_EXE]), dvd(100.0, c[WARP_E])),
                                  dvd(100.0, c[WARP_NP_E]));
        ratio = dvd(c[INST_F32 + ((k < B_ISSUE) ? (k - B_FP32) : 0)], fitted);
    }
    double r[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) r[j] = __shfl_sync(0xffffffffu, ratio, B_FP32 + j);
    if (k == B_ISSUE) {
        if (degenerate) return 0.0;
        double util_max = r[0];
#pragma unroll
        for (int j = 1; j < 7; ++j) util_max = pymax(util_max, r[j]);
        return clamp01(dvd(mul(util_max, sub(100.0, c[INST_ISSUE_U])), 100.0));
    }
    if (k >= B_FP32 && k < B_ISSUE) {
        if (degenerate) return 0.0;
        double util;
        if (generation == 0) {
            util = dvd(c[INST_ISSUE_U], 100.0);
        } else {
            const double u = dvd(c[INST_ISSUE_U], 50.0);
            util = (u < 1.0) ? u : 1.0;
        }
        return clamp01(mul(ratio, util));
    }
    return analyze_component(c, k, generation, cores, global_threads, degenerate);
}
#endif

// analyze(): c = 23 counters, generation 0 = pre_volta, 1 = volta_plus.
// Returns the degenerate_instructions flag.
CT_HD bool analyze(const double* c, int generation, int64_t cores, int64_t global_threads,
                   double* b) {
    const bool degenerate = degenerate_of(c);
    for (int k = 0; k < N_COMP; ++k)
        b[k] = analyze_component(c, k, generation, cores, global_threads, degenerate);
    return degenerate;
}

// react() value of key k (react()'s insertion order == component order).
CT_HD double react_component(double b, int k, double inst_reaction, double issue_sign) {
    if (k <= B_LOCAL) return clamp_signed(-b);
    if (k <= B_ISSUE) {
        double scaled = (b <= inst_reaction)
                            ? 0.0
                            : dvd(-sub(b, inst_reaction), sub(1.0, inst_reaction));
        if (k == B_ISSUE) scaled = mul(issue_sign, fabs(scaled));
        return clamp_signed(scaled);
    }
    return clamp_signed(b);                           // SM_E, GLOBAL_THREADS
}

CT_HD void react(const double* b, double inst_reaction, double issue_sign, double* delta) {
    for (int k = 0; k < N_COMP; ++k) delta[k] = react_component(b[k], k, inst_reaction, issue_sign);
}

}  // namespace ct

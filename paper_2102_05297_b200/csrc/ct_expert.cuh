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
// Warp form (lane k evaluates component k, all 32 lanes call it converged).
// analyze_component branches by component kind, so a warp would run the
// kinds' divisions one after another.  Here every lane runs the same three
// division stages on its own operands (lanes without a division in a stage
// divide 1 by 1); the operands are chosen with selects, so each lane performs
// exactly analyze_component's operations in its order -- bit-identical:
//   stage 1  memory: share = part / total (0 if total <= 0); tex: TEX_U / 10;
//            local: LOC_O / 100; instruction classes + issue: 100 / WARP_E,
//            100 / WARP_NP_E, ISSUE_U / 100 (pre-Volta) or / 50; SM:
//            (100 - SM_E) / 100; paral: (sat - threads) / sat
//   stage 2  memory: (share * util) / 10; local: (. * busiest) / 10;
//            classes: c / fitted
//   stage 3  issue: (util_max * (100 - ISSUE_U)) / 100 over the seven class
//            ratios taken from lanes 8..14 by shuffle
__device__ __forceinline__ double analyze_component_warp(const double* c, int k, int generation,
                                                         int64_t cores, int64_t global_threads,
                                                         bool degenerate) {
    const bool mem = k < B_TEX, tex = k == B_TEX, loc = k == B_LOCAL;
    const bool cls = (k >= B_FP32) && (k < B_ISSUE), iss = k == B_ISSUE;
    const bool inst = cls || iss;
    const bool smk = k == B_SM, par = k == B_PARAL;
    const int rd = (k < 2) ? DRAM_RT : (k < 4 ? L2_RT : SHR_LT);
    const int util_i = (k < 2) ? DRAM_U : (k < 4 ? L2_U : SHR_U);
    const double tot = mem ? add(c[rd], c[rd + 1]) : 1.0;
    const double sat = (double)(cores * 5);
    // ---- stage 1
    double n1 = 1.0, d1 = 1.0;
    if (mem) { n1 = c[rd + (k & 1)]; d1 = tot; }
    if (tex) { n1 = c[TEX_U]; d1 = 10.0; }
    if (loc) { n1 = c[LOC_O]; d1 = 100.0; }
    if (inst) { n1 = 100.0; d1 = c[WARP_E]; }
    if (smk) { n1 = sub(100.0, c[SM_E_]); d1 = 100.0; }
    if (par) { n1 = sub(sat, (double)global_threads); d1 = sat; }
    const double n2 = inst ? 100.0 : 1.0, d2 = inst ? c[WARP_NP_E] : 1.0;
    const double n3 = inst ? c[INST_ISSUE_U] : 1.0;
    const double d3 = inst ? (generation == 0 ? 100.0 : 50.0) : 1.0;
    const double q1 = dvd(n1, d1), q2 = dvd(n2, d2), q3 = dvd(n3, d3);
    // ---- stage 2
    const double share = (mem && !(tot > 0.0)) ? 0.0 : q1;       // _traffic_share
    const double busiest = pymax(pymax(c[DRAM_U], c[L2_U]), c[TEX_U]);
    const double fitted = mul(mul(mul(32.0, c[INST_EXE]), q1), q2);
    double n4 = 1.0, d4 = 1.0;
    if (mem) { n4 = mul(share, c[util_i]); d4 = 10.0; }
    if (loc) { n4 = mul(q1, busiest); d4 = 10.0; }
    if (inst) { n4 = c[INST_F32 + (cls ? k - B_FP32 : 0)]; d4 = fitted; }
    const double q4 = dvd(n4, d4);
    // ---- stage 3 (b_issue): the class ratios of lanes 8..14
    const double ratio = (cls && !degenerate) ? q4 : 0.0;
    double r[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) r[j] = __shfl_sync(0xffffffffu, ratio, B_FP32 + j);
    double util_max = r[0];
#pragma unroll
    for (int j = 1; j < 7; ++j) util_max = pymax(util_max, r[j]);
    const double q5 = dvd(iss ? mul(util_max, sub(100.0, c[INST_ISSUE_U])) : 1.0, iss ? 100.0 : 1.0);
    // ---- per-kind result
    double v;
    if (mem || loc) v = q4;
    else if (tex || smk) v = q1;
    else if (par) v = q1 > 0.0 ? q1 : 0.0;                        // max(0.0, par)
    else if (cls) {
        if (degenerate) return 0.0;
        const double util = (generation == 0) ? q3 : (q3 < 1.0 ? q3 : 1.0);
        v = mul(q4, util);
    } else {                                                      // b_issue
        if (degenerate) return 0.0;
        v = q5;
    }
    return clamp01(v);
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

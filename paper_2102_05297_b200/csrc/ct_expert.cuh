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

// analyze(): c = 23 counters, generation 0 = pre_volta, 1 = volta_plus.
// Returns the degenerate_instructions flag.
CT_HD bool analyze(const double* c, int generation, int64_t cores, int64_t global_threads,
                   double* b) {
    double rw = add(c[DRAM_RT], c[DRAM_WT]);
    b[B_DRAM_READ] = dvd(mul(share(c[DRAM_RT], rw), c[DRAM_U]), 10.0);
    b[B_DRAM_WRITE] = dvd(mul(share(c[DRAM_WT], rw), c[DRAM_U]), 10.0);
    double l2 = add(c[L2_RT], c[L2_WT]);
    b[B_L2_READ] = dvd(mul(share(c[L2_RT], l2), c[L2_U]), 10.0);
    b[B_L2_WRITE] = dvd(mul(share(c[L2_WT], l2), c[L2_U]), 10.0);
    double sh = add(c[SHR_LT], c[SHR_WT]);
    b[B_SHARED_READ] = dvd(mul(share(c[SHR_LT], sh), c[SHR_U]), 10.0);
    b[B_SHARED_WRITE] = dvd(mul(share(c[SHR_WT], sh), c[SHR_U]), 10.0);
    b[B_TEX] = dvd(c[TEX_U], 10.0);
    double busiest = pymax(pymax(c[DRAM_U], c[L2_U]), c[TEX_U]);
    b[B_LOCAL] = dvd(mul(dvd(c[LOC_O], 100.0), busiest), 10.0);

    bool degenerate = c[INST_EXE] <= 0.0 || c[WARP_E] <= 0.0 || c[WARP_NP_E] <= 0.0;
    if (degenerate) {
        for (int k = B_FP32; k <= B_ISSUE; ++k) b[k] = 0.0;
    } else {
        double fitted = mul(mul(mul(32.0, c[INST_EXE]), dvd(100.0, c[WARP_E])),
                            dvd(100.0, c[WARP_NP_E]));
        double util;
        if (generation == 0) {
            util = dvd(c[INST_ISSUE_U], 100.0);
        } else {
            double u = dvd(c[INST_ISSUE_U], 50.0);
            util = (u < 1.0) ? u : 1.0;                       // min(1.0, u)
        }
        double util_max = 0.0;
        for (int k = 0; k < 7; ++k) {
            double ratio = dvd(c[INST_F32 + k], fitted);
            b[B_FP32 + k] = mul(ratio, util);
            util_max = (k == 0) ? ratio : pymax(util_max, ratio);
        }
        b[B_ISSUE] = dvd(mul(util_max, sub(100.0, c[INST_ISSUE_U])), 100.0);
    }
    b[B_SM] = dvd(sub(100.0, c[SM_E_]), 100.0);
    double sat = (double)(cores * 5);
    double par = dvd(sub(sat, (double)global_threads), sat);
    b[B_PARAL] = par > 0.0 ? par : 0.0;                       // max(0.0, par)
    for (int k = 0; k < N_COMP; ++k) b[k] = clamp01(b[k]);
    return degenerate;
}

// react(): delta[k] for the k-th key of react()'s insertion order.
CT_HD void react(const double* b, double inst_reaction, double issue_sign, double* delta) {
    for (int k = 0; k <= B_LOCAL; ++k) delta[k] = clamp_signed(-b[k]);
    for (int k = B_FP32; k <= B_ISSUE; ++k) {
        double v = b[k];
        double scaled = (v <= inst_reaction)
                            ? 0.0
                            : dvd(-sub(v, inst_reaction), sub(1.0, inst_reaction));
        if (k == B_ISSUE) scaled = mul(issue_sign, fabs(scaled));
        delta[k] = clamp_signed(scaled);
    }
    delta[B_SM] = clamp_signed(b[B_SM]);
    delta[B_PARAL] = clamp_signed(b[B_PARAL]);
}

}  // namespace ct

// hostcheck.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the device headers' __host__ __device__ arithmetic (RNG, expert
// system, pow8, fixed point, certified selection) for the CPU so that
// tests/test_hostcheck.py can compare them with the reference in this
// container, where there is no GPU.  The product never loads this library;
// it exists so that the exact code the kernels run is pinned before it ever
// reaches a B200.  hc_profile_search() replays the kernel's per-repetition
// algorithm sequentially (same decisions: exact prefix, certification,
// sequential re-decision) to pin trajectory parity on the CPU.
#include <stdint.h>
#include <string.h>
#include <vector>

#include "countertune_b200.h"
#include "ct_expert.cuh"
#include "ct_rng.cuh"

using namespace ct;

extern "C" {

void hc_seed_pool(const uint32_t* ent, int n_ent, const uint32_t* pre, int n_pre, int has_child,
                  uint32_t child, uint32_t* out4) {
    SeedWords sw{ent, n_ent, pre, n_pre, has_child != 0, child};
    SeedPool p = seed_pool(sw);
    for (int i = 0; i < 4; ++i) out4[i] = p.w[i];
}

// ops: 0 -> integers(arg), 1 -> random(); results as double
void hc_rng_stream(const uint32_t* ent, int n_ent, const uint32_t* pre, int n_pre, int has_child,
                   uint32_t child, const int* ops, const int64_t* args, int n, double* out) {
    SeedWords sw{ent, n_ent, pre, n_pre, has_child != 0, child};
    Pcg64 g;
    g.seed(seed_pool(sw));
    for (int i = 0; i < n; ++i)
        out[i] = ops[i] == 0 ? (double)g.integers((uint64_t)args[i]) : g.next_double();
}

void hc_permutation(const uint32_t* ent, int n_ent, const uint32_t* pre, int n_pre, int has_child,
                    uint32_t child, int64_t n, int64_t* out) {
    SeedWords sw{ent, n_ent, pre, n_pre, has_child != 0, child};
    Pcg64 g;
    g.seed(seed_pool(sw));
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    for (int64_t i = n - 1; i > 0; --i) {
        int64_t j = (int64_t)g.interval((uint64_t)i);
        int64_t t = out[i]; out[i] = out[j]; out[j] = t;
    }
}

int hc_analyze(const double* c23, int generation, int64_t cores, int64_t threads, double* b18) {
    return analyze(c23, generation, cores, threads, b18) ? 1 : 0;
}

void hc_react(const double* b18, double inst_reaction, double issue_sign, double* d18) {
    react(b18, inst_reaction, issue_sign, d18);
}

void hc_pow8(const double* x, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = pow8(x[i]);
}

void hc_weights(const double* raw, const uint8_t* pool, int64_t n, double s_max, double s_min,
                double gamma, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = pool[i] ? weight(raw[i], s_max, s_min, gamma) : 0.0;
}

// fixed-point round trip helpers: returns 0 when a weight is not representable
int hc_fx_roundtrip(const double* w, int64_t n, double* back, double* floor_back) {
    int ok = 1;
    for (int64_t i = 0; i < n; ++i) {
        u128 f;
        if (!to_fx(w[i], &f)) { ok = 0; back[i] = -1.0; }
        else back[i] = fx_to_double(f);
        floor_back[i] = fx_to_double(floor_fx(w[i]));
    }
    return ok;
}

// exact sum of weights, rounded once
double hc_fx_sum(const double* w, int64_t n) {
    u128 s = 0;
    for (int64_t i = 0; i < n; ++i) { u128 f; if (to_fx(w[i], &f)) s += f; }
    return fx_to_double(s);
}

static int64_t seq_select(const double* w, int64_t n, double u) {
    double c = 0.0;
    for (int64_t i = 0; i < n; ++i) c = add(c, w[i]);
    double r = mul(u, c);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { s = add(s, w[i]); if (s > r) return i; }
    return n;
}

// certified selection on the exact prefix (same decision as warp_locate +
// certify); *cert = 1 if certified.
int64_t hc_select(const double* w, int64_t n, double u, int* cert) {
    u128 total = 0;
    std::vector<u128> f(n);
    for (int64_t i = 0; i < n; ++i) {
        if (!to_fx(w[i], &f[i])) { *cert = 0; return seq_select(w, n, u); }
        total += f[i];
    }
    double total_d = fx_to_double(total);
    double r = mul(u, total_d);
    u128 r_fx = floor_fx(r);
    u128 run = 0;
    int64_t idx = -1;
    u128 before = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (run + f[i] > r_fx) { idx = i; before = run; break; }
        run += f[i];
    }
    if (idx >= 0) {
        double bound = (double)(2 * n + 16) * 1.1102230246251565e-16 * total_d;
        u128 b_fx = floor_fx(bound) + 1;
        u128 lo = r_fx - before;
        u128 hi = before + f[idx] - r_fx - 1;
        if (lo > b_fx && hi > b_fx) { *cert = 1; return idx; }
    }
    *cert = 0;
    return seq_select(w, n, u);
}

// One repetition of the batched kernel's algorithm, sequentially.
// table: column-major (C x n).  Returns the CT_STATUS_* code; -1 error.
int hc_profile_search(const double* table, int64_t n, const double* runtime,
                      const int64_t* threads, const double* counters, const uint8_t* has_record,
                      const uint8_t* stop, const ct_search_params* prm, const uint32_t* ent,
                      int n_ent, const uint32_t* pre, int n_pre, int has_child, uint32_t child,
                      int32_t* out_idx, uint8_t* out_prof, int64_t* n_steps, int64_t* uncertified,
                      int64_t* scored) {
    SeedWords sw{ent, n_ent, pre, n_pre, has_child != 0, child};
    Pcg64 rng;
    rng.seed(seed_pool(sw));
    std::vector<uint8_t> expl(n, 0);
    std::vector<double> w(n, 0.0);
    int64_t n_expl = 0, ns = 0;
    *uncertified = 0;
    *scored = 0;
    int64_t c_prof = (int64_t)rng.integers((uint64_t)n);
    int status = CT_STATUS_BUDGET;
    for (int it = 0; it < prm->outer_iterations; ++it) {
        if (!has_record[c_prof]) { status = -1; break; }
        out_idx[ns] = (int32_t)c_prof; out_prof[ns] = 1; ++ns;
        if (!expl[c_prof]) { expl[c_prof] = 1; ++n_expl; }
        if (stop && stop[c_prof]) { status = CT_STATUS_STOPPED; break; }
        double b[N_COMP], d[N_COMP];
        analyze(counters + c_prof * N_REQ, prm->generation, prm->cores, threads[c_prof], b);
        react(b, prm->inst_reaction, prm->issue_delta_sign, d);
        ActiveTerm act[N_COMP];
        int na = 0;
        for (int k = 0; k < N_COMP; ++k) {
            if (d[k] == 0.0 || prm->delta_columns[k] < 0) continue;
            double pv = table[prm->delta_columns[k] * n + c_prof];
            if (pv == 0.0) continue;
            act[na].col = prm->delta_columns[k]; act[na].nz = 0; act[na].d = d[k]; act[na].p = pv; ++na;
        }
        if (n_expl >= n) { status = CT_STATUS_EXHAUSTED; break; }
        *scored += n - n_expl;
        double smax = -INFINITY, smin = INFINITY;
        for (int64_t e = 0; e < n; ++e) {
            if (expl[e]) { w[e] = 0.0; continue; }
            double raw = 0.0;
            for (int k = 0; k < na; ++k)
                raw = add(raw, raw_term(table[act[k].col * n + e], act[k], prm->literal_sign != 0));
            w[e] = raw;
            smax = (raw > smax || raw != raw) ? raw : smax;
            smin = (raw < smin || raw != raw) ? raw : smin;
        }
        int positive = 0;
        for (int64_t e = 0; e < n; ++e) {
            w[e] = expl[e] ? 0.0 : weight(w[e], smax, smin, prm->gamma);
            positive += w[e] > 0.0;
        }
        double t_best = INFINITY;
        bool done = false;
        for (int k = 0; k < prm->inner_steps; ++k) {
            if (positive <= 0) { status = CT_STATUS_EXHAUSTED; done = true; break; }
            double u = rng.next_double();
            int cert = 0;
            int64_t chosen = hc_select(w.data(), n, u, &cert);
            if (!cert) ++*uncertified;
            if (chosen < 0 || chosen >= n || !has_record[chosen]) { status = -1; done = true; break; }
            w[chosen] = 0.0;
            --positive;
            double rt = runtime[chosen];
            out_idx[ns] = (int32_t)chosen; out_prof[ns] = 0; ++ns;
            if (!expl[chosen]) { expl[chosen] = 1; ++n_expl; }
            if (stop && stop[chosen]) { status = CT_STATUS_STOPPED; done = true; break; }
            if (rt <= t_best) { t_best = rt; c_prof = chosen; }
        }
        if (done) break;
    }
    *n_steps = ns;
    return status;
}

}  // extern "C"

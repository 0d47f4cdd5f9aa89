// ct_models.cuh -- batched model inference: the PredictionTable of a whole
// space (search.py:54-63 over ModelSet.predict, models.py:310-333).
//
// One thread per (configuration, counter).  A tree column walks the
// flattened tree (assignment[feature] <= threshold goes left, models.py:
// 86-90); a regression column finds the model of the configuration's binary
// subspace by binary search over the column's sorted keys and sums its terms
// left to right in the reference's operation order (models.py:107-121):
//     intercept  t += c          lin    t += c * a
//     quad       t += (c * v) * v      cross  t += c * (a * b)
// then clamps at 0 as max(0.0, value) does.  A configuration whose subspace
// has no model gets 0 (the reference omits the counter; the table stores 0).
// Integer comparisons and IEEE _rn arithmetic only: the table is bit-identical
// to the reference's.
#pragma once
#include "ct_hd.cuh"

namespace ct {

struct ModelProgramDev {
    int32_t n_cols, n_params, n_binary;
    const int32_t* node_feature;
    const int32_t* node_left;
    const int32_t* node_right;
    const double* node_threshold;
    const double* node_value;
    const int32_t* col_root;
    const int32_t* col_model_first;
    const int32_t* col_model_count;
    const uint64_t* model_key;
    const int32_t* model_term_first;
    const int32_t* model_term_count;
    const int32_t* term_kind;
    const int32_t* term_p1;
    const int32_t* term_p2;
    const double* term_coef;
    const int32_t* binary_pos;
};

__device__ __forceinline__ double model_value(const ModelProgramDev& m, const double* row, int c,
                                              bool* present) {
    *present = true;
    int node = m.col_root[c];
    if (node >= 0) {
        while (m.node_feature[node] >= 0) {
            const int f = m.node_feature[node];
            node = (row[f] <= m.node_threshold[node]) ? m.node_left[node] : m.node_right[node];
        }
        return m.node_value[node];
    }
    uint64_t key = 0;
    for (int b = 0; b < m.n_binary; ++b) key = (key << 1) | (row[m.binary_pos[b]] == 1.0 ? 1u : 0u);
    int lo = m.col_model_first[c], hi = lo + m.col_model_count[c];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (m.model_key[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo >= m.col_model_first[c] + m.col_model_count[c] || m.model_key[lo] != key) {
        *present = false;
        return 0.0;
    }
    double t = 0.0;
    const int t0 = m.model_term_first[lo], t1 = t0 + m.model_term_count[lo];
    for (int k = t0; k < t1; ++k) {
        const double coef = m.term_coef[k];
        switch (m.term_kind[k]) {
        case 0: t = add(t, coef); break;
        case 1: t = add(t, mul(coef, row[m.term_p1[k]])); break;
        case 2: { const double v = row[m.term_p1[k]]; t = add(t, mul(mul(coef, v), v)); break; }
        default: t = add(t, mul(coef, mul(row[m.term_p1[k]], row[m.term_p2[k]]))); break;
        }
    }
    return t;
}

// out_rowmajor[i * n_cols + c] and the column-major device table
// table[c * ld + i] (both optional).
__global__ void k_model_predict(const ModelProgramDev m, const double* assign, int64_t n,
                                double* out_rowmajor, double* table, int64_t ld) {
    const int64_t total = n * (int64_t)m.n_cols;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        // consecutive threads take consecutive configurations of one column:
        // coalesced column-major stores, the tree walk is warp-uniform near
        // the root
        const int c = (int)(k / n);
        const int64_t i = k - (int64_t)c * n;
        bool present;
        double v = model_value(m, assign + (size_t)i * m.n_params, c, &present);
        v = (v > 0.0) ? v : 0.0;                 // max(0.0, value); NaN -> 0
        if (!present) v = 0.0;
        if (out_rowmajor) out_rowmajor[(size_t)i * m.n_cols + c] = v;
        if (table) table[(size_t)c * ld + i] = v;
    }
}

}  // namespace ct

// ct_rng.cuh -- numpy's Generator(PCG64) stream, bit for bit, host+device.
//
// The reference draws every random number from np.random.default_rng(seed)
// with seed = SeedSequence(master).spawn(R)[rep] (harness.py:135-136,
// search.py:321,359).  The stream never depends on the data, so
// each repetition regenerates it on the device from the master entropy
// alone:
//   SeedSequence mixing  -- numpy/random/bit_generator.pyx (SeedSequence:
//                           mix_entropy, generate_state; numpy 2.3, pool 4)
//   PCG64 seeding/step   -- numpy/random/src/pcg64 (pcg64_set_seed; 128-bit
//                           LCG + XSL-RR output)
//   integers(0, N)       -- buffered bounded Lemire on next_uint32 (N <= 2^32)
//   random()             -- (next_uint64 >> 11) * 2^-53
//   permutation(N)       -- Fisher-Yates from the back with random_interval
// Verified bit-exact against numpy in tests/test_hostcheck.py.
#pragma once
#include "ct_hd.cuh"

namespace ct {

// ----------------------------------------------------------- SeedSequence
struct SeedPool { uint32_t w[4]; };

CT_HD uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
    v ^= *hc;
    *hc *= 0x931e8875u;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

CT_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    r ^= r >> 16;
    return r;
}

// Assembled entropy = run entropy (zero-padded to 4 words when a spawn key
// follows) ++ spawn key words; then the pool is mixed.  `word(i)` yields the
// i-th assembled word, `n` their count.
template <typename WordFn>
CT_HD SeedPool ss_pool(WordFn word, int n) {
    SeedPool p;
    uint32_t hc = 0x43b0d7e5u;
    for (int i = 0; i < 4; ++i) p.w[i] = ss_hashmix(i < n ? word(i) : 0u, &hc);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) p.w[d] = ss_mix(p.w[d], ss_hashmix(p.w[s], &hc));
    for (int s = 4; s < n; ++s) {
        uint32_t h = 0;
        for (int d = 0; d < 4; ++d) {
            h = ss_hashmix(word(s), &hc);
            p.w[d] = ss_mix(p.w[d], h);
        }
    }
    return p;
}

// SeedSequence(entropy, spawn_key=prefix (+ child)) pool.
struct SeedWords {
    const uint32_t* entropy; int n_entropy;
    const uint32_t* prefix; int n_prefix;
    bool has_child; uint32_t child;
    CT_HD int run_len() const {
        int spawn = n_prefix + (has_child ? 1 : 0);
        return (spawn > 0 && n_entropy < 4) ? 4 : n_entropy;
    }
    CT_HD int count() const { return run_len() + n_prefix + (has_child ? 1 : 0); }
    CT_HD uint32_t operator()(int i) const {
        int rl = run_len();
        if (i < rl) return i < n_entropy ? entropy[i] : 0u;
        i -= rl;
        if (i < n_prefix) return prefix[i];
        return child;
    }
};

CT_HD SeedPool seed_pool(const SeedWords& sw) { return ss_pool(sw, sw.count()); }

// generate_state(n_words) over the mixed pool.
CT_HD void ss_generate(const SeedPool& p, uint32_t* out, int n_words) {
    uint32_t hc = 0x8b51f9ddu;
    for (int i = 0; i < n_words; ++i) {
        uint32_t v = p.w[i & 3];
        v ^= hc;
        hc *= 0x58f38dedu;
        v *= hc;
        v ^= v >> 16;
        out[i] = v;
    }
}

// ------------------------------------------------------------------ PCG64
struct Pcg64 {
    u128 state, inc;
    uint32_t has32, u32;

    CT_HD static u128 mult() {
        return (((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull;
    }
    CT_HD void step() { state = state * mult() + inc; }

    CT_HD void seed(const SeedPool& p) {
        uint32_t w[8];
        ss_generate(p, w, 8);
        uint64_t v0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        uint64_t v1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
        uint64_t v2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
        uint64_t v3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
        u128 initstate = ((u128)v0 << 64) | v1;
        u128 initseq = ((u128)v2 << 64) | v3;
        state = 0;
        inc = (initseq << 1) | 1u;
        step();
        state += initstate;
        step();
        has32 = 0;
        u32 = 0;
    }

    // XSL-RR output of a state
    CT_HD static uint64_t output(u128 s) {
        uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
        uint64_t x = hi ^ lo;
        unsigned rot = (unsigned)(hi >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }

    CT_HD uint64_t next64() {
        step();
        return output(state);
    }

    // Jump-ahead: k steps map state s to A_k s + C_k inc with A_k = M^k,
    // C_k = M^(k-1) + ... + 1 (mod 2^128); jump_tables fills k = 0..kmax.
    CT_HD static void jump_tables(u128* A, u128* C, int kmax) {
        A[0] = 1; C[0] = 0;
        for (int k = 0; k < kmax; ++k) { A[k + 1] = A[k] * mult(); C[k + 1] = C[k] * mult() + 1; }
    }
    // Generator.random() that the (k)th next call would return, k = 1, 2, ...
    CT_HD double double_after(u128 Ak, u128 Ck) const {
        return (double)(output(Ak * state + Ck * inc) >> 11) * (1.0 / 9007199254740992.0);
    }
    CT_HD void advance(u128 Ak, u128 Ck) { state = Ak * state + Ck * inc; }

    CT_HD uint32_t next32() {
        if (has32) { has32 = 0; return u32; }
        uint64_t n = next64();
        has32 = 1;
        u32 = (uint32_t)(n >> 32);
        return (uint32_t)n;
    }

    // Generator.random()
    CT_HD double next_double() {
        return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
    }

    // Generator.integers(0, n) for 1 <= n <= 2^32 (int64 dtype path:
    // random_bounded_uint64_fill -> buffered_bounded_lemire_uint32).
    CT_HD uint64_t integers(uint64_t n) {
        uint64_t rng = n - 1;
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        uint32_t rexcl = (uint32_t)(rng + 1);
        uint64_t m = (uint64_t)next32() * rexcl;
        uint32_t left = (uint32_t)m;
        if (left < rexcl) {
            uint32_t threshold = (uint32_t)((0xFFFFFFFFu - (uint32_t)rng) % rexcl);
            while (left < threshold) {
                m = (uint64_t)next32() * rexcl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }

    // random_interval(max) (Fisher-Yates index draw of Generator.shuffle).
    CT_HD uint64_t interval(uint64_t mx) {
        if (mx == 0) return 0;
        uint64_t mask = mx;
        mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
        mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
        uint64_t v;
        if (mx <= 0xFFFFFFFFull) {
            while ((v = (next32() & mask)) > mx) {}
        } else {
            while ((v = (next64() & mask)) > mx) {}
        }
        return v;
    }
};

}  // namespace ct

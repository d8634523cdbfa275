// Vectors with 2^CL < n <= 8 * 2^CL (config 2's 2^15 < n <= 2^16 lives here)
// are G = ceil(n / 2^CL) chunks of 2^CL words; chunk g = positions
// [g 2^CL, (g+1) 2^CL).  A transform touches HBM once each way (BASELINE.md
// §5 passes_min = 1).  The top gam = ceil_lg(n) - CL stages pair words in
// different chunks: per column c (stride 2^CL) they are a 2^gam-point network.
//
// Forward (k_clg_fwd, one G-CTA cluster per vector, no DSMEM): CTA g reads
// the G rows of its columns from global memory (the vector's first reader
// brings them from HBM, the others hit L2), evaluates only row g's cone of
// each column network, then the CL stages local to its chunk (sub-block g of
// the network: twiddles omega_{2J} at global J).  A split cluster barrier
// keeps every chunk store behind all siblings' row reads (in place).
//
// Inverse (K = n >> CL complete chunks, h = n mod 2^CL), split in two
// launches, k_cli_chunks then k_cli_cols:
//   1. chunks g < K: inverse of the CL local stages (left scaled by 2^CL);
//      chunk K: phase 1 of its masked inverse;
//   2. columns c >= h: K known outputs -> K coefficients by V_K^-1 (REDC
//      dot products; results straight to the vector), and the column's next
//      output sum_j x_j omega_K^j into chunk K's slot c (shared memory);
//   3. chunk K: generalised in-tile inverse with h known outputs and the
//      2^CL - h values from step 2 as its known tail;
//   4. columns c < h: K+1 known outputs -> coefficients by V_{K+1}^-1.
// The large path (n > 8 2^CL) uses the same split as two passes over HBM.
// This is the two-level form of the inverse; values equal the
// reference's Algorithm 2 because the inverse map is unique.
#pragma once
#include <cooperative_groups.h>


#include "kernels.cuh"
#include <type_traits>

// CTAs per SM the 256-thread tile kernels are compiled for: 3 (80 registers)
// for u32 words; u64 words need twice the registers per 32-word unit, so 2
template <class F>
constexpr int kern_minb() { return sizeof(typename F::W) == 8 ? 2 : 3; }

namespace cg = cooperative_groups;

// split cluster barrier (every thread of the CTA arrives / waits)
TFT_DEV void cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
TFT_DEV void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// read-only load of one twiddle pair
template <typename W>
TFT_DEV Tw<W> ldg_tw(const Tw<W>* p) {
    if constexpr (sizeof(W) == 4) {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        return Tw<W>{t.x, t.y};
    } else {
        const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(p));
        return Tw<W>{t.x, t.y};
    }
}

// N consecutive twiddle pairs from an N-aligned index (true for every call in
// reg_fwd / reg_inv), 16-byte loads
template <typename W, int N>
TFT_DEV void ldg_tw_run(const Tw<W>* p, Tw<W>* out) {
    if constexpr (sizeof(W) == 4 && N >= 2) {
#pragma unroll
        for (int q = 0; q < N; q += 2) {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(p + q));
            out[q] = Tw<W>{t.x, t.y};
            out[q + 1] = Tw<W>{t.z, t.w};
        }
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) out[q] = ldg_tw(p + q);
    }
}

// N consecutive single-word (Montgomery) twiddles -> Tw pairs {wR, wR p^-1},
// 16-byte loads where N allows (runs are N-aligned)
template <int N>
TFT_DEV void ldg_word_run(const uint32_t* p, uint32_t pinv, Tw<uint32_t>* out) {
    if constexpr (N >= 4) {
#pragma unroll
        for (int q = 0; q < N; q += 4) {
            const uint4 t = __ldg(reinterpret_cast<const uint4*>(p + q));
            out[q] = Tw<uint32_t>{t.x, t.x * pinv};
            out[q + 1] = Tw<uint32_t>{t.y, t.y * pinv};
            out[q + 2] = Tw<uint32_t>{t.z, t.z * pinv};
            out[q + 3] = Tw<uint32_t>{t.w, t.w * pinv};
        }
    } else if constexpr (N == 2) {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
        out[0] = Tw<uint32_t>{t.x, t.x * pinv};
        out[1] = Tw<uint32_t>{t.y, t.y * pinv};
    } else {
        const uint32_t w = __ldg(p);
        out[0] = Tw<uint32_t>{w, w * pinv};
    }
}

// TwDirect over the single-word table (F30M twiddles)
struct TwDirectM {
    const uint32_t* ZM;
    uint32_t blk;
    int T;
    uint32_t pinv;
    TFT_DEV Tw<uint32_t> get(int s, uint32_t J) const {
        const uint32_t w = __ldg(ZM + ((blk << (T - s - 1)) + J));
        return Tw<uint32_t>{w, w * pinv};
    }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<uint32_t>* out) const {
        ldg_word_run<N>(ZM + ((blk << (T - s - 1)) + J0), pinv, out);
    }
};

// TwBig over the single-word tables: above 2^zb the product of the two
// Montgomery words is one REDC (mont(hR, lR) = hlR), its companion one IMAD
template <class FM>
struct TwBigM {
    const uint32_t* ZM;
    const uint32_t* ZhM;
    uint64_t blk;
    int T, zb;
    FM f;
    TFT_DEV Tw<uint32_t> get(int s, uint32_t J) const {
        Tw<uint32_t> t[1];
        get_many<1>(s, J, t);
        return t[0];
    }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<uint32_t>* out) const {
        const uint64_t idx = (blk << (T - s - 1)) + J0;
        const uint64_t m = (1ull << zb) - 1;
        ldg_word_run<N>(ZM + (idx & m), f.pinv, out);
        if (idx > m) {
            const uint32_t hi = __ldg(ZhM + (idx >> zb));
#pragma unroll
            for (int q = 0; q < N; ++q) {
                const uint32_t w = f.red1(f.mont(hi, out[q].w));
                out[q] = Tw<uint32_t>{w, w * f.pinv};
            }
        }
    }
};

// Direct twiddles for a tile that is block `blk` at level T:
// theta(s, J) = omega_{2 (blk 2^(T-s-1) + J)} from the 2^zb-entry table.
// ZM: the same table as single Montgomery words; the bottom (SLO = 0) rounds
// of a Shoup field use it (their twiddles are per thread), so providers for
// F30 that reach the rounds must carry it.
template <class F>
struct TwDirect {
    static constexpr bool kMont = true;
    const Tw<typename F::W>* Z;
    uint32_t blk;
    int T;
    F f;
    const typename F::W* ZM = nullptr;
    TFT_DEV TwDirectM mont() const { return TwDirectM{(const uint32_t*)ZM, blk, T, (uint32_t)f.pinv}; }
    TFT_DEV Tw<typename F::W> get(int s, uint32_t J) const { return ldg_tw(Z + ((blk << (T - s - 1)) + J)); }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<typename F::W>* out) const {
        ldg_tw_run<typename F::W, N>(Z + ((blk << (T - s - 1)) + J0), out);
    }
};

// Twiddles for a tile that is block `blk` (64-bit) at level T of an arbitrarily
// long transform: theta(s, J) = omega_{2 idx}, idx = blk 2^(T-s-1) + J.  Below
// 2^zb the table is read directly; above, idx = hi*2^zb + lo and
// omega_{2 idx} = Zh[hi] * Z[lo] (product rule) costs one twiddle product and
// one companion.  N-aligned runs of N <= 2^zb indices never straddle a 2^zb
// boundary.
template <class F>
struct TwBig {
    static constexpr bool kMont = true;
    const Tw<typename F::W>* Z;
    const Tw<typename F::W>* Zh;
    uint64_t blk;
    int T, zb;
    F f;
    const typename F::W* ZM = nullptr;  // single-word tables (see TwDirect)
    const typename F::W* ZhM = nullptr;
    TFT_DEV TwBigM<F> mont() const { return TwBigM<F>{(const uint32_t*)ZM, (const uint32_t*)ZhM, blk, T, zb, f}; }
    TFT_DEV Tw<typename F::W> get(int s, uint32_t J) const {
        const uint64_t idx = (blk << (T - s - 1)) + J;
        const uint64_t m = (1ull << zb) - 1;
        if (idx <= m) return ldg_tw(Z + idx);
        return f.tw(f.twmul(ldg_tw(Zh + (idx >> zb)), ldg_tw(Z + (idx & m))));
    }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<typename F::W>* out) const {
        const uint64_t idx = (blk << (T - s - 1)) + J0;
        const uint64_t m = (1ull << zb) - 1;
        ldg_tw_run<typename F::W, N>(Z + (idx & m), out);
        if (idx > m) {
            const Tw<typename F::W> hi = ldg_tw(Zh + (idx >> zb));
#pragma unroll
            for (int q = 0; q < N; ++q) out[q] = f.tw(f.twmul(hi, out[q]));
        }
    }
};

// ------------------------------------------------------ compile-time rounds
// A tile of 2^TL rows x 2^WLOG interleaved columns, element (pos, col) at
// index (pos << WLOG) | col, physical slot idx + idx/32.  A unit is 2^KK
// words of one column at rows base + i 2^SLO.  Its physical offsets are
// compile-time constants in every case the round schedule produces (SLO = 0
// or SLO >= 5):
//   SLO+WLOG >= 5          : i (2^(SLO+WLOG) + 2^(SLO+WLOG-5))
//   SLO = 0, KK+WLOG <= 5  : i 2^WLOG         (unit inside one 32-word row)
//   SLO = 0, KK+WLOG > 5   : i 2^WLOG + (i >> (5-WLOG))
template <int SLO, int WLOG, int KK>
TFT_DEV constexpr uint32_t unit_off(int i) {
    return (SLO + WLOG >= 5) ? (uint32_t)i * ((1u << (SLO + WLOG)) + (1u << (SLO + WLOG - 5)))
           : (KK + WLOG <= 5) ? ((uint32_t)i << WLOG)
                              : (((uint32_t)i << WLOG) + ((uint32_t)i >> (5 - WLOG)));
}

// Forward round.  With PRUNE, units whose every output row is >= lim are
// skipped (only rows < lim are needed after the remaining stages).
template <class F, int TL, int KK, int SLO, int WLOG, bool PRUNE, int ZT = 0, class TP>
TFT_DEV void fwd_round_units(const F& f, typename F::W* S, const TP& tp, uint32_t need, Lanes ln) {
    using W = typename F::W;
    constexpr uint32_t NU = 1u << (TL - KK + WLOG);
    const uint32_t lim = PRUNE ? ((need + (1u << SLO) - 1) >> SLO) << SLO : 0;
    for (uint32_t g = ln.id; g < NU; g += ln.n) {
        const uint32_t col = g & ((1u << WLOG) - 1), u = g >> WLOG;
        const uint32_t base = (u & ((1u << SLO) - 1)) | ((u >> SLO) << (SLO + KK));
        if (PRUNE && base >= lim) continue;
        const uint32_t idx0 = (base << WLOG) | col;
        W* pb = S + idx0 + (idx0 >> 5);
        W v[1 << KK];
#pragma unroll
        for (int i = 0; i < (1 << KK); ++i)
            if (ZT == 0 || !((i >> (KK - 1)) & 1)) v[i] = pb[unit_off<SLO, WLOG, KK>(i)];  // (zero rows: not read)
        reg_fwd<F, KK, KK - 1, ZT>(f, v, base, SLO, tp);
        if constexpr (is_wide<F>::value) {
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i) v[i] = f.narrow(v[i]);
        }
#pragma unroll
        for (int i = 0; i < (1 << KK); ++i) pb[unit_off<SLO, WLOG, KK>(i)] = v[i];
    }
}

// Inverse round (stages ascending).  MASK: only pairs inside complete binary
// blocks of [0, h) run, each block scaled at its last stage (tile.cuh
// reg_inv); SCALE=false leaves an unmasked tile scaled by 2^TL.
template <class F, int TL, int KK, int SLO, int WLOG, bool MASK, bool SCALE, class TP>
TFT_DEV void inv_round_units(const F& f, typename F::W* S, const TP& tp, const Tw<typename F::W>* ipow2,
                             uint32_t h, Lanes ln) {
    using W = typename F::W;
    constexpr uint32_t NU = 1u << (TL - KK + WLOG);
    const uint32_t h_lo = MASK ? (uint32_t)(((uint64_t)h >> (SLO + 1)) << (SLO + 1)) : 0;
    const uint32_t h_top = MASK ? (uint32_t)(((uint64_t)h >> (SLO + KK)) << (SLO + KK)) : 0;
    const uint32_t h_top1 = MASK ? (uint32_t)(((uint64_t)h >> (SLO + KK + 1)) << (SLO + KK + 1)) : 0;
    for (uint32_t g = ln.id; g < NU; g += ln.n) {
        const uint32_t col = g & ((1u << WLOG) - 1), u = g >> WLOG;
        const uint32_t base = (u & ((1u << SLO) - 1)) | ((u >> SLO) << (SLO + KK));
        if (MASK && base >= h_lo) continue;
        const uint32_t idx0 = (base << WLOG) | col;
        W* pb = S + idx0 + (idx0 >> 5);
        W v[1 << KK];
#pragma unroll
        for (int i = 0; i < (1 << KK); ++i) v[i] = pb[unit_off<SLO, WLOG, KK>(i)];
        if constexpr (MASK) {
            // a unit whose aligned 2^(SLO+KK) block lies below the top stage's
            // bound is unmasked at every stage of the round; it is scaled (at
            // the top stage only) when its block closes a complete block of [0, h)
            constexpr int STOP = SLO + KK - 1;
            const uint32_t blo = (base >> (STOP + 1)) << (STOP + 1), bhi = blo + (1u << (STOP + 1));
            if (bhi <= h_top) {
                reg_inv<F, KK, 0, false>(f, v, base, SLO, tp, h, blo >= h_top1 ? STOP : -1, ipow2);
            } else {
                reg_inv<F, KK, 0, true>(f, v, base, SLO, tp, h, -1, ipow2);
            }
        } else {
            reg_inv<F, KK, 0, false>(f, v, base, SLO, tp, h, SCALE ? TL - 1 : -1, ipow2);
        }
        if constexpr (is_wide<F>::value) {
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i) v[i] = f.narrow(v[i]);
        }
        if constexpr (MASK) {
            // only rows < h change; the rest is not written back
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i)
                if (base + ((uint32_t)i << SLO) < h) pb[unit_off<SLO, WLOG, KK>(i)] = v[i];
        } else {
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i) pb[unit_off<SLO, WLOG, KK>(i)] = v[i];
        }
    }
}

// In the bottom round (SLO = 0) every thread needs its own 2^KK - 1
// twiddles -- about one per tile word, more bytes than the tile itself in
// 8-byte pairs.  For u32 words that round reads the single-word tables
// instead: Montgomery words whose companion is one IMAD.  For p < 2^32 the
// product is unchanged (F32 is Montgomery already); for p < 2^30 it becomes
// F30M's Montgomery product (one more IMAD.HI than Shoup per butterfly).
template <class F, class TP>
__host__ __device__ constexpr bool bottom_words() {
    if constexpr (std::is_same<F, F30>::value || std::is_same<F, F32>::value) return TP::kMont;
    else return false;
}
template <class F>
TFT_DEV auto bottom_field(const F& f) {
    if constexpr (std::is_same<F, F30>::value) return F30M(f);
    else if constexpr (std::is_same<F, F32>::value) return F32W(f);
    else return f;
}
// the field a register round computes in: F32 rounds run on wide words
// (field.cuh F32W) and narrow them when the unit is written back
template <class F>
TFT_DEV auto round_field(const F& f) {
    if constexpr (std::is_same<F, F32>::value) return F32W(f);
    else return f;
}

template <class F, int TL, int KK, int SLO, int WLOG, bool PRUNE, int ZT = 0, class TP>
TFT_DEV void fwd_round_ct(const F& f, typename F::W* S, const TP& tp, uint32_t need, Lanes ln) {
    if constexpr (SLO == 0 && WLOG == 0 && bottom_words<F, TP>()) {
        const auto fb = bottom_field(f);
        fwd_round_units<decltype(fb), TL, KK, SLO, WLOG, PRUNE, ZT>(fb, S, tp.mont(), need, ln);
    } else {
        const auto fr = round_field(f);
        fwd_round_units<decltype(fr), TL, KK, SLO, WLOG, PRUNE, ZT>(fr, S, tp, need, ln);
    }
}

template <class F, int TL, int KK, int SLO, int WLOG, bool MASK, bool SCALE, class TP>
TFT_DEV void inv_round_ct(const F& f, typename F::W* S, const TP& tp, const Tw<typename F::W>* ipow2,
                          uint32_t h, Lanes ln) {
    if constexpr (SLO == 0 && WLOG == 0 && bottom_words<F, TP>()) {
        const auto fb = bottom_field(f);
        inv_round_units<decltype(fb), TL, KK, SLO, WLOG, MASK, SCALE>(fb, S, tp.mont(), ipow2, h, ln);
    } else {
        const auto fr = round_field(f);
        inv_round_units<decltype(fr), TL, KK, SLO, WLOG, MASK, SCALE>(fr, S, tp, ipow2, h, ln);
    }
}

// stages [0, SHI): one round of min(5, SHI-5) stages from the top (s_lo >= 5),
// recursing down to a final 5-or-fewer-stage round at s_lo = 0.
// ZT (first call only, SHI = TL): rows >= 2^(TL-ZT) of the tile are zero on
// entry; the top round's first ZT layers are copies (clamped to that round).
template <class F, int TL, int SHI, int WLOG = 0, bool PRUNE = false, int ZT = 0, class TP>
TFT_DEV void fwd_rounds_ct(const F& f, typename F::W* S, const TP& tp, uint32_t need = 0, Lanes ln = cta_lanes()) {
    if constexpr (SHI <= 5) {
        fwd_round_ct<F, TL, SHI, 0, WLOG, PRUNE, (ZT < SHI ? ZT : SHI)>(f, S, tp, need, ln);
        __syncthreads();
    } else {
        constexpr int KK = (SHI - 5) >= 5 ? 5 : (SHI - 5);
        fwd_round_ct<F, TL, KK, SHI - KK, WLOG, PRUNE, (ZT < KK ? ZT : KK)>(f, S, tp, need, ln);
        __syncthreads();
        fwd_rounds_ct<F, TL, SHI - KK, WLOG, PRUNE>(f, S, tp, need, ln);
    }
}

template <class F, int TL, int SHI, bool MASK, class TP, bool SCALE = true, int WLOG = 0>
TFT_DEV void inv_rounds_ct(const F& f, typename F::W* S, const TP& tp, const Tw<typename F::W>* ipow2,
                           uint32_t h = 0, Lanes ln = cta_lanes()) {
    if constexpr (SHI <= 5) {
        inv_round_ct<F, TL, SHI, 0, WLOG, MASK, SCALE>(f, S, tp, ipow2, h, ln);
        __syncthreads();
    } else {
        constexpr int KK = (SHI - 5) >= 5 ? 5 : (SHI - 5);
        inv_rounds_ct<F, TL, SHI - KK, MASK, TP, SCALE, WLOG>(f, S, tp, ipow2, h, ln);
        inv_round_ct<F, TL, KK, SHI - KK, WLOG, MASK, SCALE>(f, S, tp, ipow2, h, ln);
        __syncthreads();
    }
}

// dot product of M canonical words with M Montgomery words, reduced once:
// the raw 64-bit products accumulate exactly while their sum stays below
// p 2^32 (<= 4 terms for p < 2^30), then one REDC gives the value
TFT_DEV uint32_t redc_dot4(const F30& f, const uint32_t* y, const uint32_t* wM, int m) {
    uint64_t acc = 0;
#pragma unroll 4
    for (int c = 0; c < 4; ++c)
        if (c < m) acc += (uint64_t)y[c] * wM[c];
    const uint32_t q = (uint32_t)acc * f.npinv;
    return f.red1((uint32_t)((acc + (uint64_t)q * f.p) >> 32));
}

// Constants of the small-network column solves (F30): the row scale
// s = 2^-CL of the split inverse's chunk pass, s/2, s/4, 1/2, 1/4, the
// point w = omega_2 = Z[1] (omega_0..3 = 1, -1, w, -w), s w^-1 / 4, w^-1 / 4.
struct SmallNet {
    Tw<uint32_t> s, s2, s4, h2, h4, w, swi4, wi4;
};

// The column solve for M <= 4 known outputs as the inverse of the 4-point
// column network on 1, -1, w, -w, instead of the dense V_M^-1: 3-5 Shoup
// products instead of M^2 (+ M for the next output).  Rows are scaled by
// 2^CL except, with LASTS, the last one (the split inverse's convention,
// vinvS / vinvT).  Outputs canonical; the next output F(omega_M) for M < 4.
template <int M, bool LASTS>
TFT_DEV void col_solve_net(const F30& f, const uint32_t* y, const SmallNet& k, uint32_t* xv, uint32_t* nv) {
    const uint32_t p = f.p, p2 = f.p2;
    if constexpr (M == 1) {
        const uint32_t x0 = f.canon(f.mulw(y[0], k.s));
        xv[0] = x0;
        if (nv) *nv = x0;
    } else if constexpr (M == 2) {
        uint32_t x0, x1;
        if constexpr (!LASTS) {
            x0 = f.mulw(y[0] + y[1], k.s2);
            x1 = f.mulw(y[0] - y[1] + p, k.s2);
        } else {
            const uint32_t c0 = f.mulw(y[0], k.s);
            x0 = f.mulw(c0 + y[1], k.h2);
            x1 = f.mulw(c0 - y[1] + p, k.h2);
        }
        xv[0] = f.canon(x0);
        xv[1] = f.canon(x1);
        if (nv) *nv = f.canon(x0 + f.mulw(x1, k.w));  // F(w) = x0 + w x1
    } else if constexpr (M == 3) {
        const uint32_t a1 = f.mulw(y[0] - y[1] + p, k.s2);  // x1
        const uint32_t t = f.mulw(a1, k.w);
        const uint32_t c2 = LASTS ? y[2] : f.mulw(y[2], k.s);
        const uint32_t a2 = f.red2(c2 - t + p2);            // x0 - x2
        const uint32_t m = f.mulw(y[0] + y[1], k.s4), q = f.mulw(a2, k.h2);
        xv[0] = f.canon(m + q);
        xv[1] = f.canon(a1);
        xv[2] = f.canon(m - q + p2);
        if (nv) *nv = f.canon(a2 - t + p2);                 // F(-w) = (x0 - x2) - w x1
    } else {
        static_assert(M == 4, "small column networks have at most 4 points");
        const uint32_t P = y[0] + y[1], Q = y[0] - y[1] + p;
        uint32_t x0, x2, m2;
        if constexpr (!LASTS) {
            x0 = f.mulw(P + y[2] + y[3], k.s4);
            x2 = f.mulw(P - (y[2] + y[3]) + p2, k.s4);  // (P, y2 + y3 < 2p: no wrap)
            m2 = f.mulw(y[2] - y[3] + p, k.swi4);
        } else {
            const uint32_t c2 = f.mulw(y[2], k.s);
            const uint32_t u = f.mulw(P, k.s4), v = f.mulw(c2 + y[3], k.h4);
            x0 = u + v;
            x2 = u - v + p2;
            m2 = f.mulw(c2 - y[3] + p, k.wi4);
        }
        const uint32_t m1 = f.mulw(Q, k.s4);
        xv[0] = f.canon(x0);
        xv[1] = f.canon(m1 + m2);
        xv[2] = f.canon(x2);
        xv[3] = f.canon(m1 - m2 + p2);
    }
}

// column solve: y[0..M) are the column's first M outputs; xv <- its M
// coefficients (V_M^-1, M^2 products, canonical) and, if wanted, nv <- the
// next output sum_j x_j omega_M^j.  With sn (F30, M <= 4; M = 4 without a
// next output) the small-network solve above replaces the dense products.
template <class F, int M, bool LASTS = false>
TFT_DEV void col_solve_vals(const F& f, const typename F::W* yin, const Tw<typename F::W>* blk,
                            const typename F::W* blkM, typename F::W* xv, typename F::W* nv,
                            const SmallNet* sn = nullptr) {
    using W = typename F::W;
    W y[M];
#pragma unroll
    for (int j = 0; j < M; ++j) y[j] = f.canon(yin[j]);
    if constexpr (std::is_same<F, F30>::value && M <= 4) {
        if (sn && !(M == 4 && nv)) {
            col_solve_net<M, LASTS>(f, y, *sn, xv, nv);
            return;
        }
    }
    if constexpr (std::is_same<F, F30>::value) {
        // REDC dot products over raw Montgomery entries, <= 4 terms per reduction
#pragma unroll
        for (int r = 0; r < M; ++r) {
            W acc = redc_dot4(f, y, blkM + 8 * r, M);  // canonical
#pragma unroll
            for (int c0 = 4; c0 < M; c0 += 4) acc = f.cadd(acc, redc_dot4(f, y + c0, blkM + 8 * r + c0, M - c0));
            xv[r] = acc;
        }
    } else {
#pragma unroll
        for (int r = 0; r < M; ++r) {
            W acc = 0;
#pragma unroll
            for (int c = 0; c < M; ++c) acc = f.cadd(acc, f.cmulw(y[c], blk[8 * r + c]));
            xv[r] = acc;
        }
    }
    if (nv) {
        W acc = 0;
        if constexpr (std::is_same<F, F30>::value) {
            acc = redc_dot4(f, xv, blkM + 64, M);
#pragma unroll
            for (int c0 = 4; c0 < M; c0 += 4) acc = f.cadd(acc, redc_dot4(f, xv + c0, blkM + 64 + c0, M - c0));
        } else {
#pragma unroll
            for (int c = 0; c < M; ++c) acc = f.cadd(acc, f.cmulw(xv[c], blk[64 + c]));
        }
        *nv = acc;
    }
}

// solve columns [lo, hi): ld(j, c) gives row j < M of column c (DSMEM or
// global); the M coefficients of a column are final outputs and go straight
// to the vector in global memory (row r of column c is x[r C + c]; a warp's
// stores are 32 consecutive words); with write_next the next output goes to
// nx(c, value)
template <class F, int M, bool LASTS = false, class LD, class NX>
TFT_DEV void col_solve_range(const F& f, const LD& ld, const NX& nx, typename F::W* xg, uint32_t C, uint32_t lo,
                             uint32_t hi, const Tw<typename F::W>* blk, const typename F::W* blkM,
                             bool write_next, const SmallNet* sn = nullptr) {
    using W = typename F::W;
    uint32_t c = lo + threadIdx.x;
    auto one = [&](uint32_t cc, const W* y) {
        W xv[M], nv;
        col_solve_vals<F, M, LASTS>(f, y, blk, blkM, xv, write_next ? &nv : nullptr, sn);
#pragma unroll
        for (int r = 0; r < M; ++r) xg[(size_t)r * C + cc] = xv[r];
        if (write_next) nx(cc, nv);
    };
    // CIF columns per thread: CIF*M loads in flight before any math
    constexpr int CIF = M <= 2 ? 8 : (M <= 4 ? 4 : 2);
    for (; c + (CIF - 1) * blockDim.x < hi; c += CIF * blockDim.x) {
        W y[CIF][M];
#pragma unroll
        for (int k = 0; k < CIF; ++k)
#pragma unroll
            for (int j = 0; j < M; ++j) y[k][j] = ld(j, c + k * blockDim.x);
#pragma unroll
        for (int k = 0; k < CIF; ++k) one(c + k * blockDim.x, y[k]);
    }
    for (; c < hi; c += blockDim.x) {
        W y[M];
#pragma unroll
        for (int j = 0; j < M; ++j) y[j] = ld(j, c);
        one(c, y);
    }
}

// Column solve over columns [clo, chi) of a vector laid out as rows of C
// words: M = KG + (LASTS ? 1 : 0) known rows, rows j < KG from global memory
// (x[j C + c]) and, with LASTS, row KG from the tile S; the M coefficients
// go back to x rows 0..M-1 and, with NEXT, the column's next output to S[c].
// u32 words: 4 adjacent columns per thread with 16-byte loads and stores
// (rows share the vector's alignment, C being a multiple of 4), ragged edges
// through col_solve_range.
template <class F, int M, bool LASTS, bool NEXT>
TFT_DEV void colq_solve(const F& f, typename F::W* x, typename F::W* S, uint32_t C, uint32_t clo, uint32_t chi,
                        const Tw<typename F::W>* blk, const typename F::W* blkM, const SmallNet* sn = nullptr) {
    using W = typename F::W;
    constexpr int KG = LASTS ? M - 1 : M, QIF = M <= 3 ? 2 : 1;
    auto ld = [&](int j, uint32_t c) { return j < KG ? __ldcg(x + (size_t)j * C + c) : S[c + (c >> 5)]; };
    auto nx = [&](uint32_t c, W w) { S[c + (c >> 5)] = w; };
    if (clo >= chi) return;
    if constexpr (M > 4 || sizeof(W) != 4) {  // (few vectors; registers would spill) scalar loads
        col_solve_range<F, M, LASTS>(f, ld, nx, x, C, clo, chi, blk, blkM, NEXT, sn);
        return;
    }
    const uint32_t mis = (uint32_t)(((uintptr_t)(x + clo) & 15) / sizeof(W));
    const uint32_t head = min(chi - clo, (4 - mis) & 3);
    const uint32_t c_a = clo + head, nq = (chi - c_a) / 4, c_b = c_a + 4 * nq;
    if (head) col_solve_range<F, M, LASTS>(f, ld, nx, x, C, clo, c_a, blk, blkM, NEXT, sn);
    for (uint32_t q0 = threadIdx.x; q0 < nq; q0 += QIF * blockDim.x) {
        uint4 r[QIF][KG];
#pragma unroll
        for (int u = 0; u < QIF; ++u) {
            const uint32_t c0 = c_a + 4 * (q0 + u * blockDim.x);
#pragma unroll
            for (int j = 0; j < KG; ++j)
                if (q0 + u * blockDim.x < nq) r[u][j] = __ldcg(reinterpret_cast<const uint4*>(x + (size_t)j * C + c0));
        }
#pragma unroll
        for (int u = 0; u < QIF; ++u) {
            const uint32_t c0 = c_a + 4 * (q0 + u * blockDim.x);
            if (q0 + u * blockDim.x >= nq) break;
            W out[M][4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                W y[M], xv[M], nv;
#pragma unroll
                for (int j = 0; j < KG; ++j) y[j] = k == 0 ? r[u][j].x : k == 1 ? r[u][j].y : k == 2 ? r[u][j].z : r[u][j].w;
                const uint32_t c = c0 + k;
                if (LASTS) y[M - 1] = S[c + (c >> 5)];
                col_solve_vals<F, M, LASTS>(f, y, blk, blkM, xv, NEXT ? &nv : nullptr, sn);
                if (NEXT) S[c + (c >> 5)] = nv;
#pragma unroll
                for (int j = 0; j < M; ++j) out[j][k] = xv[j];
            }
#pragma unroll
            for (int j = 0; j < M; ++j)
                *reinterpret_cast<uint4*>(x + (size_t)j * C + c0) = make_uint4(out[j][0], out[j][1], out[j][2], out[j][3]);
        }
    }
    if (c_b < chi) col_solve_range<F, M, LASTS>(f, ld, nx, x, C, c_b, chi, blk, blkM, NEXT, sn);
}

// Split inverse for 2^CL < n <= 8 2^CL (no cluster): two launches.
// A (k_cli_chunks, grid (G, vectors)): complete chunks g < K run their
//   inverse rounds (left scaled by 2^CL) and the last chunk the masked phase
//   1 of its solve; each stores its tile back as is.
// B (k_cli_cols, one CTA per vector): columns >= h solved from the K
//   complete rows (coefficients final; each column's next output into the
//   last chunk's tail, in shared memory), then phases 2/3 of the last
//   chunk and the columns < h from K + 1 rows.
// Every CTA works alone, so nothing waits on a sibling; the price is one
// more read and write of the vector (the in-between state stays in the
// n-word buffer: no scratch).
// B: the column solves and the last chunk's phases 2/3 of vector v (rows
// read through L2: in the fused launch they were written moments ago)
template <class F, int CL>
TFT_DEV void cli_cols_body(const LaunchArgs<F>& a, int64_t v, typename F::W* S, bool prefetch) {
    using W = typename F::W;
    constexpr uint32_t C = 1u << CL;
    const int64_t n = a.xd.n(v);
    const uint32_t K = (uint32_t)(n >> CL), h = (uint32_t)(n & (C - 1));
    W* x = a.x + a.xd.o(v);
    const F f = a.f;
    // stream the vector into L2 (TMA bulk prefetch) while the first quads load
    if (prefetch && threadIdx.x == 0) l2_prefetch(x, n);
    const Tw<W>* b1 = a.R.vinvS + 72 * (K - 1);
    const W* b1M = a.R.vinvM + 8 * 72 + 72 * (K - 1);
    // small-network solves (F30): the scale and point constants, per thread
    SmallNet snv{};
    const SmallNet* sn = nullptr;
    if constexpr (std::is_same<F, F30>::value) {
        const Tw<W>* ip = a.R.ipow2;
        snv = SmallNet{ip[CL], ip[CL + 1], ip[CL + 2], ip[1], ip[2], a.R.Zf[1],
                       f.tw(f.twmul(a.R.Zi[1], ip[CL + 2])), f.tw(f.twmul(a.R.Zi[1], ip[2]))};
        if (!a.dense_cols) sn = &snv;
    }
    switch (K) {  // columns >= h: K rows
#define TFTB_C1(k)                                                                          \
    case k:                                                                                 \
        if (h) colq_solve<F, k, false, true>(f, x, S, C, h, C, b1, b1M, sn);                \
        else colq_solve<F, k, false, false>(f, x, S, C, 0, C, b1, b1M, sn);                 \
        break;
        TFTB_C1(1) TFTB_C1(2) TFTB_C1(3) TFTB_C1(4) TFTB_C1(5) TFTB_C1(6) TFTB_C1(7)
        default: colq_solve<F, 8, false, false>(f, x, S, C, 0, C, b1, b1M); break;  // K = 8: h = 0
#undef TFTB_C1
    }
    if (!h) return;
    // the last chunk's known outputs [0, h) (its tail [h, C) came from the
    // column solve above: no zero fill)
    tile_load<W>(S, x + (size_t)K * C, h, h, [](uint32_t, W w) { return w; });
    __syncthreads();
    const TwDirect<F> tpi{a.R.Zi, K, CL, f, a.R.ZiM};
    itft_phases23<0>(f, SmemTile<W>{S, CL, 0}, h, TwDirect<F>{a.R.Zf, K, CL, f}, tpi, a.R);
    const Tw<W>* b2 = a.R.vinvT + 72 * K;
    const W* b2M = a.R.vinvM + 16 * 72 + 72 * K;
    switch (K + 1) {  // columns < h: K + 1 rows, the last from the tile
#define TFTB_C2(m)                                                                          \
    case m: colq_solve<F, m, true, false>(f, x, S, C, 0, h, b2, b2M, sn); break;
        TFTB_C2(2) TFTB_C2(3) TFTB_C2(4) TFTB_C2(5) TFTB_C2(6) TFTB_C2(7) TFTB_C2(8)
#undef TFTB_C2
    }
}

// A (and, fused, B): chunk g of vector v runs its inverse rounds and stores
// the tile back.  With a.done (the production path) the vector's chunk CTAs
// then take a ticket, and the LAST one to finish runs B for the vector
// right away: no second launch, no CTA ever waits on a sibling, and the
// rows B reads were written microseconds earlier, so they come from L2
// (and the first, intermediate write of each row is usually overwritten
// there before it reaches HBM).  Tickets are self-resetting.
template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_cli_chunks(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    const uint32_t g = blockIdx.x;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const uint32_t K = (uint32_t)(n >> CL), h = (uint32_t)(n & (C - 1));
    const int64_t cbase = (int64_t)g * C;
    if (cbase >= n) return;
    const int64_t o = a.xd.o(v);
    W* x = a.x + o;
    const F f = a.f;
    if (a.pre)
        tile_load_pre<F>(a, S, x + cbase, a.pre + o + cbase, n - cbase, C);
    else
        tile_load<W>(S, x + cbase, n - cbase, C, [](uint32_t, W w) { return w; });
    __syncthreads();
    const TwDirect<F> tpi{a.R.Zi, g, CL, f, a.R.ZiM};
    if (g < K) inv_rounds_ct<F, CL, CL, false, TwDirect<F>, false>(f, S, tpi, a.R.ipow2);
    else inv_rounds_ct<F, CL, CL, true>(f, S, tpi, a.R.ipow2, h);
    const uint32_t lim = (uint32_t)min((int64_t)C, n - cbase);
    if (!a.done) {
        tile_store<W>(x + cbase, S, lim, [](W w) { return w; });
        return;
    }
    const auto id = [](W w) { return w; };
    tile_store<W, decltype(id), false>(x + cbase, S, lim, id);
    __shared__ unsigned last;
    __threadfence();  // this CTA's rows, visible device-wide before its ticket
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned chunks = K + (h ? 1u : 0u);
        const unsigned t = atomicAdd(a.done + (v - a.vbase), 1u);
        last = t == chunks - 1;
        if (last) a.done[v - a.vbase] = 0;  // reset for the next execution
    }
    __syncthreads();
    if (!last) return;
    __threadfence();  // acquire: the siblings' rows
    cli_cols_body<F, CL>(a, v, S, false);
}

template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_cli_cols(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    cli_cols_body<F, CL>(a, a.vbase + blockIdx.x, S, true);
}

// ================================================ two-pass plan, chunk pass
// Chunks are 2^CL contiguous words = sub-block k of the network at level CL;
// twiddles come from TwBig (block k).  grid: (max chunks, vectors).
template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_chunk_fwd(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const uint32_t k = blockIdx.x;
    const int64_t cbase = (int64_t)k * C;
    if (cbase >= n) return;
    const F f = a.f;
    W* x = a.x + a.xd.o(v) + cbase;
    const W* st = a.stash + (v - a.vbase) * (int64_t)C;
    const int64_t avail = n - cbase;
    tile_load<W>(S, x, avail, C, [&](uint32_t i, W w) { return (int64_t)i < avail ? w : st[i]; });
    __syncthreads();
    fwd_rounds_ct<F, CL, CL, 0, true>(f, S, TwBig<F>{a.R.Zf, a.R.Zfh, k, CL, a.R.zb, f, a.R.ZfM, a.R.ZfhM},
                                      (uint32_t)min((int64_t)C, avail));
    tile_store<W>(x, S, (uint32_t)min((int64_t)C, avail), [&](W w) { return f.canon(w); });
}

// step 1: complete chunks k < K, plus phase 1 of the partial chunk K (the
// masked inverse of the complete binary blocks of its h known outputs, which
// needs nothing from the columns) so the serial step 3 only runs the two
// O(2^CL) sweeps.  grid: (max chunks, vectors)
template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_chunk_inv(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const uint32_t K = (uint32_t)(n >> CL), h = (uint32_t)(n & (C - 1));
    // the partial chunk (longest CTA: masked rounds) takes block 0 so it does
    // not become the grid's tail
    const uint32_t k = !h ? blockIdx.x : (blockIdx.x == 0 ? K : blockIdx.x - 1);
    if (k > K || (k == K && !h)) return;
    const uint32_t len = k < K ? C : h;
    const F f = a.f;
    const int64_t o = a.xd.o(v) + (int64_t)k * C;
    W* x = a.x + o;
    if (a.pre)
        tile_load_pre<F>(a, S, x, a.pre + o, len, C);
    else
        tile_load<W>(S, x, len, C, [](uint32_t, W w) { return w; });
    __syncthreads();
    const TwBig<F> tpi{a.R.Zi, a.R.Zih, k, CL, a.R.zb, f, a.R.ZiM, a.R.ZihM};
    if (k < K) inv_rounds_ct<F, CL, CL, false>(f, S, tpi, a.R.ipow2);
    else inv_rounds_ct<F, CL, CL, true>(f, S, tpi, a.R.ipow2, h);
    tile_store<W>(x, S, len, [&](W w) { return f.canon(w); });
}

// step 3: the partial last chunk: its h slots already hold the phase-1
// values (k_chunk_inv); the C-h stashed inputs complete it.  grid: (1, vectors)
template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_last_inv(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const uint32_t K = (uint32_t)(n >> CL), h = (uint32_t)(n & (C - 1));
    if (!h) return;
    const F f = a.f;
    const int64_t o = a.xd.o(v) + (int64_t)K * C;
    W* x = a.x + o;
    const W* st = a.stash + (v - a.vbase) * (int64_t)C;
    TFTB_TAIL_STAMP(a, 8);
    tile_load<W>(S, x, h, C, [&](uint32_t i, W w) { return i < h ? w : st[i]; });
    __syncthreads();
    TFTB_TAIL_STAMP(a, 9);
    const TwBig<F> tpf{a.R.Zf, a.R.Zfh, K, CL, a.R.zb, f}, tpi{a.R.Zi, a.R.Zih, K, CL, a.R.zb, f};
    SmemTile<W> tl{S, CL, 0};
    itft_phases23<0>(f, tl, h, tpf, tpi, a.R);
    TFTB_TAIL_STAMP(a, 10);
    tile_store<W>(x, S, h, [&](W w) { return f.canon(w); });
    TFTB_TAIL_STAMP(a, 11);
}

// ================================================ two-pass plan, column pass
// Columns are nodes (c, l1) of the reference tree: rows r at positions
// r 2^l1 + c.  One CTA owns 2^WLOG adjacent columns of 2^L0 rows.
template <class F>
__host__ __device__ constexpr int col_tile_log() { return sizeof(typename F::W) == 4 ? 14 : 13; }
// adjacent columns per CTA: a 2^col_tile_log-word tile, at most 2^10
// columns, so short columns still fill a 64 KB tile and keep enough bytes
// in flight (= host.h make_plan's wlog)
template <class F, int L0>
__host__ __device__ constexpr int col_wlog() {
    return (col_tile_log<F>() - L0) < 0 ? 0 : ((col_tile_log<F>() - L0) > 10 ? 10 : (col_tile_log<F>() - L0));
}

// S[(r << WLOG) | col] = xf(r, col, valid ? src[r*C + col] : 0), valid = r*C + col < avail;
// 16-byte loads along rows, UNR in flight.  Every row shares the alignment
// of src (C is a multiple of the vector), so the columns [head, head + 4 nqr)
// are whole quads in every row; the few columns before and after go scalar.
template <typename W, int L0, int WLOG, int UNR = 8, class XF>
TFT_DEV void col_load(W* S, const W* src, uint32_t C, int64_t avail, const XF& xf) {
    constexpr int NV = 16 / sizeof(W);
    constexpr uint32_t R = 1u << L0, NC = 1u << WLOG;
    auto put = [&](uint32_t r, uint32_t c, W w) {
        const uint32_t idx = (r << WLOG) | c;
        S[idx + (idx >> 5)] = xf(r, c, w);
    };
    const uint32_t mis = (uint32_t)(((uintptr_t)src & 15) / sizeof(W));
    const uint32_t head = (C % NV) ? NC : min(NC, (uint32_t)((NV - mis) % NV));
    // quads per row: NC/NV when aligned, one fewer otherwise (compile-time
    // divisors either way)
    constexpr uint32_t QA = NC / NV, QM = QA > 0 ? QA - 1 : 0;
    auto quads = [&](auto nqr_c) {
        constexpr uint32_t NQR = decltype(nqr_c)::value;
        if constexpr (NQR > 0) {
            constexpr uint32_t nq = R * NQR;
            for (uint32_t q0 = threadIdx.x; q0 < nq; q0 += blockDim.x * UNR) {
                typename Vec16<W>::T buf[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t q = q0 + u * blockDim.x;
                    const uint32_t r = q / NQR, c = head + (q % NQR) * NV;
                    const int64_t pos = (int64_t)r * C + c;
                    if (q < nq && pos + NV <= avail) {
                        buf[u] = ld_stream(reinterpret_cast<const typename Vec16<W>::T*>(src + pos));
                    } else {
                        W e[NV];
#pragma unroll
                        for (int k = 0; k < NV; ++k) e[k] = (q < nq && pos + k < avail) ? src[pos + k] : W(0);
                        buf[u] = Vec16<W>::make(e);
                    }
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t q = q0 + u * blockDim.x;
                    if (q >= nq) break;
                    const uint32_t r = q / NQR, c = head + (q % NQR) * NV;
#pragma unroll
                    for (int k = 0; k < NV; ++k) put(r, c + k, Vec16<W>::get(buf[u], k));
                }
            }
        }
    };
    uint32_t tail;
    if (head == 0) {
        quads(std::integral_constant<uint32_t, QA>{});
        tail = QA * NV;
    } else if (head < NC) {
        quads(std::integral_constant<uint32_t, QM>{});
        tail = head + QM * NV;
    } else {
        tail = NC;
    }
    // the edge columns [0, head) and [tail, NC) of every row
    const uint32_t ne = head + (NC - tail);
    for (uint32_t g = threadIdx.x; g < R * ne; g += blockDim.x) {
        const uint32_t r = g / ne, j = g % ne, c = j < head ? j : tail + (j - head);
        const int64_t pos = (int64_t)r * C + c;
        put(r, c, pos < avail ? src[pos] : W(0));
    }
}

// x_t[r C + c] = canon(S[(r << WLOG) | c]) for rows [r0, r1) and tile columns
// [clo, chi) (x_t = the tile's first column in the vector).  Whole-width
// stores of 16-byte-aligned rows go out as 16-byte vectors (rows share the
// alignment of x_t: C is a multiple of the vector width); edges scalar.
// Plain stores: the other pass reads these words next, often from L2.
template <class F, int WLOG>
TFT_DEV void col_store(const F& f, typename F::W* xt, const typename F::W* S, uint32_t C, uint32_t r0, uint32_t r1,
                       uint32_t clo, uint32_t chi) {
    using W = typename F::W;
    using V = Vec16<W>;
    constexpr int NV = V::N;
    constexpr uint32_t NC = 1u << WLOG;
    if (r1 <= r0 || chi <= clo) return;
    if constexpr (NC >= (uint32_t)NV) {
        if (clo == 0 && chi == NC && ((uintptr_t)xt & 15) == 0) {
            constexpr uint32_t QR = NC / NV;  // vectors per row
            const uint32_t nq = (r1 - r0) * QR;
            for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
                const uint32_t r = r0 + q / QR, c = (q % QR) * NV;
                const uint32_t idx = (r << WLOG) | c;
                const W* s = S + idx + (idx >> 5);  // (NV words inside one padded 32-word row)
                W e[NV];
#pragma unroll
                for (int k = 0; k < NV; ++k) e[k] = f.canon(s[k]);
                *reinterpret_cast<typename V::T*>(xt + (size_t)r * C + c) = V::make(e);
            }
            return;
        }
    }
    const uint32_t w = chi - clo, cnt = (r1 - r0) * w;
    for (uint32_t g = threadIdx.x; g < cnt; g += blockDim.x) {
        const uint32_t r = r0 + g / w, c = clo + g % w;
        const uint32_t idx = (r << WLOG) | c;
        xt[(size_t)r * C + c] = f.canon(S[idx + (idx >> 5)]);
    }
}

// ZT: the input's rows >= 2^(L0-ZT) are zero padding in every column (a
// product's operand, ceil(nin / C) <= 2^(L0-ZT), checked by the host)
template <class F, int L0, int ZT = 0>
__global__ void __launch_bounds__(256) k_colc_fwd(LaunchArgs<F> a) {
    using W = typename F::W;
    constexpr int WLOG = col_wlog<F, L0>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v), nin = a.ind.n(v);
    const int l1 = a.l1;
    if (ceil_lg_dev(n) - l1 != L0) return;
    const uint32_t C = 1u << l1, c0 = blockIdx.x << WLOG;
    const uint32_t K = (uint32_t)(n >> l1), h = (uint32_t)(n & (C - 1));
    const F f = a.f;
    W* x = a.x + a.xd.o(v);
    const W* in = a.in + a.ind.o(v);
    col_load<W, L0, WLOG>(S, in + c0, C, nin - c0, [](uint32_t, uint32_t, W w) { return w; });
    __syncthreads();
    // rows <= K are the only outputs (row K: real for c < h, the stash for c >= h)
    fwd_rounds_ct<F, L0, L0, WLOG, true, ZT>(f, S, TwPrefix<F>{a.R.Zf}, K + (h ? 1u : 0u));
    const uint32_t NC = 1u << WLOG;
    // complete rows r < K, then row K: real words for c < h, the stash for c >= h
    col_store<F, WLOG>(f, x + c0, S, C, 0, min(K, 1u << L0), 0, NC);
    if (h && K < (1u << L0)) {
        W* st = a.stash + (v - a.vbase) * (int64_t)C;
        for (uint32_t col = threadIdx.x; col < NC; col += blockDim.x) {
            const uint32_t c = c0 + col, g = (K << WLOG) | col;
            const W w = f.canon(S[g + (g >> 5)]);
            if (c < h) x[(size_t)K * C + c] = w;
            else st[c] = w;
        }
    }
}

// inverse steps 2 (which = 0: columns c >= h, K rows, stash their row K) and
// 4 (which = 1: columns c < h, K+1 rows).  grid: (C >> WLOG, vectors)
template <class F, int L0>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_colc_inv(LaunchArgs<F> a, int which) {
    using W = typename F::W;
    constexpr int WLOG = col_wlog<F, L0>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const int l1 = a.l1;
    if (ceil_lg_dev(n) - l1 != L0) return;
    const uint32_t C = 1u << l1, c0 = blockIdx.x << WLOG, NC = 1u << WLOG;
    const uint32_t K = (uint32_t)(n >> l1), h = (uint32_t)(n & (C - 1));
    const uint32_t lo = which == 0 ? h : 0, hi = which == 0 ? C : h;
    if (c0 + NC <= lo || c0 >= hi) return;
    const uint32_t rows = which == 0 ? K : K + 1;
    const F f = a.f;
    W* x = a.x + a.xd.o(v);
    // the tile's row segments into L2 (TMA bulk prefetch), one per thread --
    // only when they are long (short columns, wide tiles): thousands of tiny
    // segments cost more than they hide (single 2^25-word vectors: +7%)
    if constexpr (((1u << WLOG) * sizeof(W)) >= 1024) {
        for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) {
            const int64_t b = (int64_t)r * C + c0;
            if (b < n) l2_prefetch(x + b, min((int64_t)NC, n - b));
        }
    }
    col_load<W, L0, WLOG>(S, x + c0, C, n - c0, [&](uint32_t r, uint32_t, W w) { return r < rows ? w : W(0); });
    __syncthreads();
    const TwPrefix<F> tpf{a.R.Zf}, tpi{a.R.Zi};
    inv_rounds_ct<F, L0, L0, true, TwPrefix<F>, true, WLOG>(f, S, tpi, a.R.ipow2, rows);
    SmemTile<W> tl{S, L0, WLOG};
    itft_phases23<WLOG>(f, tl, rows, tpf, tpi, a.R, cta_lanes(), false, true);
    // (every position of rows < rows in [lo, hi) is < n: row K only for c < h)
    col_store<F, WLOG>(f, x + c0, S, C, 0, rows, max(lo, c0) - c0, min(hi, c0 + NC) - c0);
    if (which == 0 && h) {
        W* red = S + padded_words(1u << (L0 + WLOG));
        W* nv = red + blockDim.x;
        colsum_pow(f, tl, K, K & (0u - K), omega_w(f, a.R, K), a.R.oneW, red, nv);  // (H = K's lowest set bit)
        for (uint32_t col = threadIdx.x; col < NC; col += blockDim.x) {
            const uint32_t c = c0 + col;
            if (c >= h) a.stash[(v - a.vbase) * (int64_t)C + c] = nv[col];
        }
    }
}

// Inverse step 2 for vectors whose last chunk is nearly full (few columns
// c >= h, e.g. n = 2^k - 1): one CTA per such column instead of one per
// 2^WLOG-column tile.  A lone tile CTA transforms 2^col_tile_log words to
// solve a handful of columns while the GPU waits for it (the steps after it
// are serial: single 2^25 - 1-word vector, 77 us); a column CTA transforms
// 2^L0.  Same arithmetic as k_colc_inv(which = 0) on that column.
// grid: (C - h, vectors), uniform lengths only (dispatch.cuh)
template <class F, int L0>
__global__ void __launch_bounds__(256) k_col1_inv(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    const int l1 = a.l1;
    if (ceil_lg_dev(n) - l1 != L0) return;
    const uint32_t C = 1u << l1;
    const uint32_t K = (uint32_t)(n >> l1), h = (uint32_t)(n & (C - 1));
    const uint32_t c = h + blockIdx.x;
    if (!h || c >= C) return;
    const F f = a.f;
    W* x = a.x + a.xd.o(v) + c;
    TFTB_TAIL_STAMP(a, 0);
    for (uint32_t r = threadIdx.x; r < (1u << L0); r += blockDim.x) S[r + (r >> 5)] = r < K ? x[(size_t)r * C] : W(0);
    __syncthreads();
    TFTB_TAIL_STAMP(a, 1);
    const TwPrefix<F> tpf{a.R.Zf}, tpi{a.R.Zi};
    inv_rounds_ct<F, L0, L0, true, TwPrefix<F>, true, 0>(f, S, tpi, a.R.ipow2, K);
    TFTB_TAIL_STAMP(a, 2);
    SmemTile<W> tl{S, L0, 0};
    itft_phases23<0>(f, tl, K, tpf, tpi, a.R, cta_lanes(), false, true);
    TFTB_TAIL_STAMP(a, 3);
    for (uint32_t r = threadIdx.x; r < K; r += blockDim.x) x[(size_t)r * C] = f.canon(S[r + (r >> 5)]);
    W* red = S + padded_words(1u << L0);
    W* nv = red + blockDim.x;
    TFTB_TAIL_STAMP(a, 4);
    colsum_pow(f, tl, K, K & (0u - K), omega_w(f, a.R, K), a.R.oneW, red, nv);  // (H = K's lowest set bit)
    if (threadIdx.x == 0) a.stash[(v - a.vbase) * (int64_t)C + c] = nv[0];
    TFTB_TAIL_STAMP(a, 5);
}

// ============================ forward for 2^CL < n <= 8 2^CL, no DSMEM
// CTA g of vector v needs row g of every column's 2^GAM-point network.  It
// reads the column's rows straight from global memory (the first CTA of a
// vector brings them from HBM, its siblings hit L2) and evaluates only the
// cone of row g: the top stage has theta = 1 (adds only), stage sp keeps the
// half selected by bit sp of g with one twiddle omega_{2 (g >> (sp+1))}, so a
// word costs at most GAM-1 products (<= 1 for config 2).  No DSMEM; grid
// (G, vectors) in clusters of G, whose only use is the split barrier that
// orders the in-place chunk stores after the siblings' row reads.
template <class F, int GAM>
TFT_DEV typename F::W cone_row(const F& f, typename F::W* vals, uint32_t g, const Tw<typename F::W>* tw) {
    using W = typename F::W;
    constexpr int GP = 1 << GAM;
    if constexpr (F::kLazy) {
        // inputs are canonical residues: the top stage (theta = 1) gives
        // [0, 2p) without a reduction, so does the second stage's left
        // operand; later stages reduce it from [0, 4p)
        {
            constexpr int H = GP / 2;
            const bool sel = (g >> (GAM - 1)) & 1;
#pragma unroll
            for (int i = 0; i < H; ++i) vals[i] = sel ? vals[i] - vals[i + H] + f.p : vals[i] + vals[i + H];
        }
#pragma unroll
        for (int sp = GAM - 2; sp >= 0; --sp) {
            const int H = 1 << sp;
            const bool sel = (g >> sp) & 1;
            const Tw<W> t = tw[sp];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const W a = sp == GAM - 2 ? vals[i] : f.red2(vals[i]);
                const W b = f.mulw(vals[i + H], t);
                vals[i] = sel ? a - b + f.p2 : a + b;
            }
        }
        return vals[0];
    }
    // top stage: theta = 1
    {
        constexpr int H = GP / 2;
        const bool sel = (g >> (GAM - 1)) & 1;
#pragma unroll
        for (int i = 0; i < H; ++i) vals[i] = f.half1(vals[i], vals[i + H], sel);
    }
#pragma unroll
    for (int sp = GAM - 2; sp >= 0; --sp) {
        const int H = 1 << sp;
        const bool sel = (g >> sp) & 1;
        const Tw<W> t = tw[sp];
#pragma unroll
        for (int i = 0; i < H; ++i) vals[i] = f.half(vals[i], vals[i + H], t, sel);
    }
    return vals[0];
}

// Row g of the cone (compile-time g: the half selections are constants),
// canonical inputs (see cone_row).
template <class F, int GAM, int GI>
TFT_DEV typename F::W cone_row_ct(const F& f, typename F::W* vals, const Tw<typename F::W>* tw) {
    using W = typename F::W;
    if constexpr (!F::kLazy) {
        return cone_row<F, GAM>(f, vals, GI, tw);
    } else {
        constexpr int GP = 1 << GAM;
        {
            constexpr int H = GP / 2;
            constexpr bool sel = (GI >> (GAM - 1)) & 1;
#pragma unroll
            for (int i = 0; i < H; ++i) vals[i] = sel ? vals[i] - vals[i + H] + f.p : vals[i] + vals[i + H];
        }
#pragma unroll
        for (int sp = GAM - 2; sp >= 0; --sp) {
            const int H = 1 << sp;
            const bool sel = (GI >> sp) & 1;
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const W a = sp == GAM - 2 ? vals[i] : f.red2(vals[i]);
                const W b = f.mulw(vals[i + H], tw[sp]);
                vals[i] = sel ? a - b + f.p2 : a + b;
            }
        }
        return vals[0];
    }
}

// S[i] <- row GI of column i's cone, i < 2^CL, reading the GP rows
// in[j 2^CL + i] (positions >= nin are zeros).  Rows share their 16-byte
// alignment: scalar head, then quads -- per row a quad is full, empty or
// (at most once per row) partial, decided on 32-bit offsets against the
// row's precomputed length -- then a scalar tail.
template <class F, int CL, int GAM, int GI, int NR = (1 << GAM)>
TFT_DEV void cone_fill(const F& f, typename F::W* S, const typename F::W* in, int64_t nin,
                       const Tw<typename F::W>* Zf) {
    using W = typename F::W;
    using V = Vec16<W>;
    constexpr uint32_t C = 1u << CL;
    constexpr int GP = 1 << GAM, NV = V::N;
    Tw<W> tw[GAM > 1 ? GAM - 1 : 1];
#pragma unroll
    for (int sp = 0; sp < GAM - 1; ++sp) tw[sp] = Zf[GI >> (sp + 1)];
    const uint32_t mis = (uint32_t)(((uintptr_t)in & 15) / sizeof(W));
    const uint32_t head = (NV - mis) % NV;
    uint32_t len[GP];  // words of row j present from position head on
#pragma unroll
    for (int j = 0; j < GP; ++j) {
        const int64_t r = nin - (int64_t)j * C - head;
        // rows >= NR (the vector has NR chunks) are known zeros at compile time
        len[j] = j >= NR || r <= 0 ? 0u : (uint32_t)min(r, (int64_t)C);
    }
    auto one = [&](uint32_t i) {
        W vals[GP];
#pragma unroll
        for (int j = 0; j < GP; ++j) vals[j] = j < NR && (int64_t)j * C + i < nin ? in[(size_t)j * C + i] : W(0);
        S[i + (i >> 5)] = cone_row_ct<F, GAM, GI>(f, vals, tw);
    };
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) one(i);
    const uint32_t nq = (C - head) / NV;
    const W* base = in + head;
    constexpr int UNR = GP <= 4 ? 2 : 1;
    // The vector's G CTAs start together and read the same rows.  Each
    // starts at its own 1/GP of the columns (rotated order), so at any
    // moment they fetch different lines: one CTA brings a line from HBM and
    // the siblings that reach it later hit it in L2, instead of all G
    // waiting on the same HBM fill in lockstep.
    const uint32_t shift = GI * (nq / GP);
    auto rot = [&](uint32_t q) { return q >= nq ? q : (q + shift < nq ? q + shift : q + shift - nq); };
    for (uint32_t q0 = threadIdx.x; q0 < nq; q0 += blockDim.x * UNR) {
        typename V::T buf[UNR][GP];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t o = rot(q0 + u * blockDim.x) * NV;
#pragma unroll
            for (int j = 0; j < GP; ++j) {
                const W* src = base + (size_t)j * C + o;
                if (o + NV <= len[j]) {
                    // the vector's other CTAs read the same rows: keep them in L2
                    buf[u][j] = __ldcg(reinterpret_cast<const typename V::T*>(src));
                } else if (o >= len[j]) {
                    buf[u][j] = V::zero();
                } else {
                    W e[NV];
#pragma unroll
                    for (int k = 0; k < NV; ++k) e[k] = o + k < len[j] ? src[k] : W(0);
                    buf[u][j] = V::make(e);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t q = q0 + u * blockDim.x;
            if (q >= nq) break;
            const uint32_t i0 = head + rot(q) * NV;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                W vals[GP];
#pragma unroll
                for (int j = 0; j < GP; ++j) vals[j] = V::get(buf[u][j], k);
                const uint32_t i = i0 + k;
                S[i + (i >> 5)] = cone_row_ct<F, GAM, GI>(f, vals, tw);
            }
        }
    }
    for (uint32_t i = head + nq * NV + threadIdx.x; i < C; i += blockDim.x) one(i);
}

// Split forward (no cluster), two launches:
// A (k_clf_cols, one CTA per vector): every column's 2^GAM-point network
//   over the G rows (one read of the vector); rows < K (complete chunks) go
//   back in place, row K (the last chunk, virtual words included) stays in
//   shared memory and is transformed right there, only its first h outputs
//   stored.  All of the vector's reads precede its writes in this one CTA.
// B (k_clf_chunks, grid (G, vectors)): complete chunks g < K run their CL
//   stages (sub-block g) on the column outputs.
// Used where the cone forward's clusters cost the most (see dispatch).
template <class F, int GAM>
TFT_DEV void col_net(const F& f, typename F::W* v, const Tw<typename F::W>* tw) {
    // v[r], r < 2^GAM: canonical inputs of one column -> outputs in [0, 4p)
    // (lazy fields) or canonical (F32).  Stage sp pairs rows (r, r + 2^sp)
    // with twiddle omega_{2 (r >> (sp+1))} = tw[r >> (sp+1)]; the top one is 1.
    using W = typename F::W;
    constexpr int GP = 1 << GAM;
#pragma unroll
    for (int sp = GAM - 1; sp >= 0; --sp) {
#pragma unroll
        for (int r = 0; r < GP; ++r) {
            if (r & (1 << sp)) continue;
            const int u = r + (1 << sp);
            if constexpr (F::kLazy) {
                if (sp == GAM - 1) {  // theta = 1 on canonical inputs: [0, 2p)
                    const W a = v[r], b = v[u];
                    v[r] = a + b;
                    v[u] = a - b + f.p;
                } else {
                    const W a = sp == GAM - 2 ? v[r] : f.red2(v[r]);
                    const W b = f.mulw(v[u], tw[r >> (sp + 1)]);
                    v[r] = a + b;
                    v[u] = a - b + f.p2;
                }
            } else {
                f.fwd(v[r], v[u], tw[r >> (sp + 1)]);
            }
        }
    }
}

template <class F, int CL, int GAM>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_clf_cols(LaunchArgs<F> a) {
    using W = typename F::W;
    using V = Vec16<W>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    constexpr int GP = 1 << GAM, NV = V::N;
    const int64_t v = a.vbase + blockIdx.x;
    const int64_t n = a.xd.n(v), nin = a.ind.n(v);
    const uint32_t K = (uint32_t)(n >> CL), h = (uint32_t)(n & (C - 1));
    const F f = a.f;
    W* x = a.x + a.xd.o(v);
    const W* in = a.in + a.ind.o(v);
    Tw<W> tw[GP / 2];
#pragma unroll
    for (int k = 0; k < GP / 2; ++k) tw[k] = a.R.Zf[k];
    uint32_t len[GP];  // words present in input row j
#pragma unroll
    for (int j = 0; j < GP; ++j) {
        const int64_t r = nin - (int64_t)j * C;
        len[j] = r <= 0 ? 0u : (uint32_t)min(r, (int64_t)C);
    }
    auto emit = [&](uint32_t c, const W* col) {
#pragma unroll
        for (int r = 0; r < GP; ++r) {
            if ((uint32_t)r < K) x[(size_t)r * C + c] = col[r];
            else if ((uint32_t)r == K && h) S[c + (c >> 5)] = col[r];
        }
    };
    auto one = [&](uint32_t c) {
        W col[GP];
#pragma unroll
        for (int j = 0; j < GP; ++j) col[j] = c < len[j] ? in[(size_t)j * C + c] : W(0);
        col_net<F, GAM>(f, col, tw);
        emit(c, col);
    };
    // input rows share the alignment of `in`, output rows that of `x`:
    // 16-byte quads where both agree (always, for a transform in place)
    const uint32_t mis_i = (uint32_t)(((uintptr_t)in & 15) / sizeof(W));
    const uint32_t mis_x = (uint32_t)(((uintptr_t)x & 15) / sizeof(W));
    const uint32_t head = mis_i == mis_x ? (NV - mis_i) % NV : C;
    for (uint32_t c = threadIdx.x; c < head; c += blockDim.x) one(c);
    const uint32_t nq = head < C ? (C - head) / NV : 0;
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const uint32_t c0 = head + q * NV;
        typename V::T buf[GP];
#pragma unroll
        for (int j = 0; j < GP; ++j) {
            const W* src = in + (size_t)j * C + c0;
            if (c0 + NV <= len[j]) {
                buf[j] = __ldcs(reinterpret_cast<const typename V::T*>(src));  // read once
            } else if (c0 >= len[j]) {
                buf[j] = V::zero();
            } else {
                W e[NV];
#pragma unroll
                for (int k = 0; k < NV; ++k) e[k] = c0 + k < len[j] ? src[k] : W(0);
                buf[j] = V::make(e);
            }
        }
        W out[GP][NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            W col[GP];
#pragma unroll
            for (int j = 0; j < GP; ++j) col[j] = V::get(buf[j], k);
            col_net<F, GAM>(f, col, tw);
#pragma unroll
            for (int r = 0; r < GP; ++r) out[r][k] = col[r];
        }
#pragma unroll
        for (int r = 0; r < GP; ++r) {
            if ((uint32_t)r < K) {
                __stcg(reinterpret_cast<typename V::T*>(x + (size_t)r * C + c0), V::make(out[r]));
            } else if ((uint32_t)r == K && h) {
#pragma unroll
                for (int k = 0; k < NV; ++k) S[(c0 + k) + ((c0 + k) >> 5)] = out[r][k];
            }
        }
    }
    for (uint32_t c = head + nq * NV + threadIdx.x; c < C && head < C; c += blockDim.x) one(c);
    if (!h) return;
    __syncthreads();
    fwd_rounds_ct<F, CL, CL, 0, true>(f, S, TwDirect<F>{a.R.Zf, K, CL, f, a.R.ZfM}, h);
    tile_store<W>(x + (size_t)K * C, S, h, [&](W w) { return f.canon(w); });
}

template <class F, int CL>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_clf_chunks(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    const uint32_t g = blockIdx.x;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v);
    if (((int64_t)g + 1) * C > n) return;  // complete chunks only
    const F f = a.f;
    W* x = a.x + a.xd.o(v) + (size_t)g * C;
    tile_load<W>(S, x, C, C, [](uint32_t, W w) { return w; });
    __syncthreads();
    fwd_rounds_ct<F, CL, CL, 0, true>(f, S, TwDirect<F>{a.R.Zf, g, CL, f, a.R.ZfM}, C);
    tile_store<W>(x, S, C, [&](W w) { return f.canon(w); });
}

template <class F, int CL, int GAM, int NR = (1 << GAM), bool TIM = false>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_clg_fwd(LaunchArgs<F> a) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    constexpr uint32_t C = 1u << CL;
    constexpr int GP = 1 << GAM;
    constexpr int NV = 16 / sizeof(W);
    const uint32_t g = blockIdx.x;
    const int64_t v = a.vbase + blockIdx.y;
    const int64_t n = a.xd.n(v), nin = a.ind.n(v);
    const int64_t cbase = (int64_t)g * C;
    if (cbase >= n) {  // (never for a plan's vectors) still takes part in the cluster barrier
        cluster_arrive_release();
        cluster_wait_acquire();
        return;
    }
    const F f = a.f;
    W* x = a.x + a.xd.o(v);
    const W* in = a.in + a.ind.o(v);
    TFTB_STAMP(a, 0);
    switch (g) {  // the cone's half selections are compile-time per CTA
        case 0: cone_fill<F, CL, GAM, 0, NR>(f, S, in, nin, a.R.Zf); break;
        case 1: cone_fill<F, CL, GAM, 1, NR>(f, S, in, nin, a.R.Zf); break;
        case 2: if constexpr (GAM >= 2) cone_fill<F, CL, GAM, 2, NR>(f, S, in, nin, a.R.Zf); break;
        case 3: if constexpr (GAM >= 2) cone_fill<F, CL, GAM, 3, NR>(f, S, in, nin, a.R.Zf); break;
        case 4: if constexpr (GAM >= 3) cone_fill<F, CL, GAM, 4, NR>(f, S, in, nin, a.R.Zf); break;
        case 5: if constexpr (GAM >= 3) cone_fill<F, CL, GAM, 5, NR>(f, S, in, nin, a.R.Zf); break;
        case 6: if constexpr (GAM >= 3) cone_fill<F, CL, GAM, 6, NR>(f, S, in, nin, a.R.Zf); break;
        default: if constexpr (GAM >= 3) cone_fill<F, CL, GAM, 7, NR>(f, S, in, nin, a.R.Zf); break;
    }
    TFTB_STAMP(a, 1);
    // In place (in == x), chunk g is also a row of every sibling CTA's
    // columns: this CTA's reads are done, and it may not overwrite its chunk
    // before every sibling has signalled the same.  The vector's G CTAs are
    // one cluster (co-scheduled), so the split barrier cannot deadlock, and
    // the rounds below hide its latency.
    cluster_arrive_release();
    __syncthreads();
    TFTB_STAMP(a, 2);
    fwd_rounds_ct<F, CL, CL, 0, true>(f, S, TwDirect<F>{a.R.Zf, g, CL, f, a.R.ZfM}, (uint32_t)min((int64_t)C, n - cbase));
    TFTB_STAMP(a, 5);
    cluster_wait_acquire();
    const uint32_t lim = (uint32_t)min((int64_t)C, n - cbase);
    tile_store<W>(x + cbase, S, lim, [&](W w) { return f.canon(w); });
    TFTB_STAMP(a, 6);
}

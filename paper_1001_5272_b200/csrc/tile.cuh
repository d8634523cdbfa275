// Shared-memory tile engine: one CTA transforms 2^wlog interleaved columns of
// 2^t words each (column-interleaved: element (pos, col) lives at index
// pos*2^wlog + col, physical slot idx + idx/32 to break power-of-two bank
// strides).
//
// Network convention (the reference's, `_kernels.pyx:181-223`): forward stage
// s pairs (u, u + 2^s) with u mod 2^(s+1) < 2^s and multiplies the upper
// element by theta = omega_{2J}, J = u >> (s+1), global stage order s = t-1
// .. 0.  A tile that is a sub-block B of a larger transform (positions
// [B*2^t, (B+1)*2^t) after the stages above it) uses omega_{2(B*2^(t-s-1)+J)};
// B = 0 is the untwisted case whose twiddles are the prefix Z[0..2^(t-1)) of
// one size-independent table.
//
// Stages run in register rounds of KK <= 5 stages: a thread loads 2^KK
// words spaced 2^s_lo apart, runs KK butterfly layers in registers and
// writes them back.  The last forward (first inverse) round always has
// s_lo = 0 so every round either has s_lo = 0 or s_lo >= 5, which keeps all
// shared-memory accesses bank-conflict free with the 1-in-32 padding.
#pragma once
#include "field.cuh"

// The threads that cooperate on one tile: the whole CTA by default, or a
// slice of it when a CTA carries several small tiles (k_tile_*).
struct Lanes {
    uint32_t id, n;
};
__device__ __forceinline__ Lanes cta_lanes() { return Lanes{threadIdx.x, blockDim.x}; }

template <typename W>
struct SmemTile {
    W* S;
    int t;     // log2 transform length (rows per column)
    int wlog;  // log2 interleaved columns
    TFT_DEV W& at(uint32_t idx) const { return S[idx + (idx >> 5)]; }
    TFT_DEV uint32_t ix(uint32_t pos, uint32_t col) const { return (pos << wlog) | col; }
    TFT_DEV uint32_t words() const { return 1u << (t + wlog); }
};

__host__ __device__ inline uint32_t padded_words(uint32_t words) { return words + (words >> 5) + 1; }

// Per-ring device tables (built once per RingConfig by the host).
template <typename W>
struct RingDev {
    const Tw<W>* Zf;    // Zf[j] = omega_{2j},      j < 2^zb
    const Tw<W>* Zi;    // Zi[j] = omega_{2j}^-1
    const Tw<W>* Zfh;   // Zfh[i] = omega_{2 i 2^zb}, i < 2^zh
    const Tw<W>* Zih;
    const Tw<W>* ipow2; // ipow2[k] = 2^-k, k < 64
    const Tw<W>* vinv;  // 8 blocks of 72: V_m^-1 (m x m, V_m[s][i] = omega_s^i), then omega_m^i
    const Tw<W>* vinvS; // same with every column times 2^-CL
    const Tw<W>* vinvT; // same with all but the last column times 2^-CL
    const W* vinvM;     // vinv, vinvS, vinvT as raw Montgomery words (3 x 8 x 72)
    const W* ZfM;       // Zf, Zi, Zfh, Zih as single Montgomery words w R mod p
    const W* ZiM;       // (Shoup fields only, else null): the bottom rounds'
    const W* ZfhM;      // per-thread twiddles at half the bytes
    const W* ZihM;
    Tw<W> inv2;         // 1/2
    W r2w;              // R^2 mod p as a raw word: mont(mont(a, b), r2w) = a b
    W oneW;             // 1 as a field word (1, or R mod p for Montgomery fields)
    int zb, zh;
};

// omega_{2J} for an arbitrary J < 2^(zb+zh), as a canonical field word.
template <class F>
TFT_DEV typename F::W zbig(const F& f, const RingDev<typename F::W>& R, uint64_t J, bool inverse) {
    const Tw<typename F::W>* lo = inverse ? R.Zi : R.Zf;
    const Tw<typename F::W>* hi = inverse ? R.Zih : R.Zfh;
    uint64_t m = (1ull << R.zb) - 1;
    if (J <= m) return lo[J].w;
    return f.twmul(hi[J >> R.zb], lo[J & m]);
}

// omega_s (modring.py:223-234) as a field word: omega_{2j+1} = -omega_{2j}.
template <class F>
TFT_DEV typename F::W omega_w(const F& f, const RingDev<typename F::W>& R, uint64_t s) {
    typename F::W w = zbig(f, R, s >> 1, false);
    return (s & 1) ? f.p - w : w;
}

// base^e for a field word base (square and multiply on twiddles)
template <class F>
TFT_DEV typename F::W pow_w(const F& f, typename F::W base, typename F::W one, uint64_t e) {
    typename F::W r = one;
    Tw<typename F::W> b = f.tw(base);
    while (e) {
        if (e & 1) r = f.twmul(f.tw(r), b);
        e >>= 1;
        if (e) b = f.tw(f.twmul(b, b));
    }
    return r;
}

// ---------------------------------------------------------------- twiddles
template <class F>
struct TwPrefix {  // untwisted tile: theta(s, J) = Z[J]
    static constexpr bool kMont = false;
    const Tw<typename F::W>* Z;
    TFT_DEV Tw<typename F::W> get(int, uint32_t J) const { return Z[J]; }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<typename F::W>* out) const {
#pragma unroll
        for (int q = 0; q < N; ++q) out[q] = Z[J0 + q];
    }
};

// ------------------------------------------------ in-register butterfly layers
// A unit holds 2^KK words v[i] at positions base + i*2^slo.  Layer ST (stage
// s = slo + ST) pairs (i, i + 2^ST) with twiddle index (base >> (s+1)) + q,
// q = i >> (ST+1).  Template recursion keeps every index a compile-time
// constant so the unit stays in registers.
// ZT: the unit's top ZT layers have an all-zero upper input (the zero padding
// of a product's operand, known to the host): (a + w 0, a - w 0) is a copy.
template <class F, int KK, int ST, int ZT = 0, class TP>
TFT_DEV void reg_fwd(const F& f, typename F::W* v, uint32_t base, int slo, const TP& tp) {
    using W = typename F::W;
    constexpr int NQ = 1 << (KK - 1 - ST);
    const int s = slo + ST;
    if constexpr (ST >= KK - ZT) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int r = 0; r < (1 << ST); ++r) {
                const int i = (q << (ST + 1)) | r;
                v[i | (1 << ST)] = v[i];
            }
    } else {
        Tw<W> w[NQ];
        tp.template get_many<NQ>(s, base >> (s + 1), w);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const Tw<W> t = w[q];
#pragma unroll
            for (int r = 0; r < (1 << ST); ++r) {
                const int i = (q << (ST + 1)) | r;
                f.fwd(v[i], v[i | (1 << ST)], t);
            }
        }
    }
    if constexpr (ST > 0) reg_fwd<F, KK, ST - 1, ZT>(f, v, base, slo, tp);
}

// ascending layers ST .. KK-1; pairs with pos >= lim[s] are skipped (MASK) and
// pairs with pos >= scl[s] (or, unmasked, the layer at s == last) are scaled
template <class F, int KK, int ST, bool MASK, class TP>
TFT_DEV void reg_inv(const F& f, typename F::W* v, uint32_t base, int slo, const TP& tp, uint32_t h, int last,
                     const Tw<typename F::W>* ipow2) {
    using W = typename F::W;
    constexpr int NQ = 1 << (KK - 1 - ST);
    const int s = slo + ST;
    Tw<W> w[NQ];
    tp.template get_many<NQ>(s, base >> (s + 1), w);
    const uint32_t hs = MASK ? (uint32_t)(((uint64_t)h >> (s + 1)) << (s + 1)) : 0;
    const uint32_t hs1 = MASK ? (uint32_t)(((uint64_t)h >> (s + 2)) << (s + 2)) : 0;
    const bool scale_all = !MASK && s == last;
    const Tw<W> sc = ipow2[s + 1];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const Tw<W> t = w[q];
        // hs and hs1 are multiples of the pair group's span 2^(s+1), so the
        // group's 2^ST pairs lie on one side of each: one test per group
        const uint32_t posq = base + ((uint32_t)(q << (ST + 1)) << slo);
        if (MASK && posq >= hs) continue;
        const bool scl = MASK ? posq >= hs1 : scale_all;
#pragma unroll
        for (int r = 0; r < (1 << ST); ++r) {
            const int i = (q << (ST + 1)) | r;
            if constexpr (is_wide<F>::value) {
                // the upper word is canonical when it comes from the tile
                // (first layer) or was the product side of the layer below
                // (bit ST-1 of its index; an active pair's sub-blocks were
                // active below, masked or not)
                f.inv(v[i], v[i | (1 << ST)], t, ST == 0 || ((r >> (ST > 0 ? ST - 1 : 0)) & 1));
            } else {
                f.inv(v[i], v[i | (1 << ST)], t);
            }
            if (scl) {
                v[i] = f.scale(v[i], sc);
                v[i | (1 << ST)] = f.scale(v[i | (1 << ST)], sc);
            }
        }
    }
    if constexpr (ST + 1 < KK) reg_inv<F, KK, ST + 1, MASK>(f, v, base, slo, tp, h, last, ipow2);
}

// Generalised in-tile inverse (every column at once): slots [0, h) hold
// transform outputs, slots [h, 2^t) hold KNOWN coefficients (zeros for a plain
// ITFT, stashed virtual values for the last chunk of a two-pass ITFT).  On
// return slots [0, h) hold the coefficients; [h, 2^t) are clobbered.
// This is van der Hoeven's recursive ITFT unrolled into three sweeps:
//   1. inverse-transform every complete binary block of [0, h) (masked rounds);
//   2. top-down over levels d (block holding h): either split known tails
//      into the right half (bit d-1 of h set) or fold them into the left half;
//   3. bottom-up: recombine the halves with one inverse butterfly.
// Same values as the reference's Algorithm 2 since the
// inverse map is unique; the odd-tail Horner passes are not needed.
//
// WL >= 0: the tile's column count 2^WL known at compile time (every caller:
// single-column tiles and chunks WL = 0, two-pass column tiles their WLOG),
// so the per-element index arithmetic folds to constants.
template <int WL = -1, class F, class TPF, class TPI>
TFT_DEV void itft_phases23(const F& f, const SmemTile<typename F::W>& tl, uint32_t h, const TPF& tpf,
                      const TPI& tpi, const RingDev<typename F::W>& R, Lanes ln = cta_lanes(),
                      bool uniform = false, bool zero_tail = false) {
    using W = typename F::W;
    const int t = tl.t;
    const int wl = WL >= 0 ? WL : tl.wlog;
    // uniform: every tile of the CTA walks all levels (the barriers must
    // match); tiles with nothing to do at a level just skip its work
    const bool act = h != 0 && h < (1u << t);
    if (!uniform && !act) return;
    const int dact = act ? __ffs(h) : t + 1;  // levels d with h mod 2^d != 0
    const int dlo = uniform ? 1 : dact;
    // (one barrier per level at a convergent point: with several tiles per
    // warp, lanes of one warp may be active at different levels).  Each
    // level's twiddle is fetched one level ahead so its global-memory latency
    // overlaps the previous level instead of sitting between two barriers.
    auto tw2 = [&](int d) {  // phase-2 twiddle of level d
        const uint32_t B = h - (h & ((1u << d) - 1));
        return tpf.get(d - 1, B >> d);
    };
    auto tw3 = [&](int d) {  // phase-3 twiddle of level d
        const uint32_t hd = h & ((1u << d) - 1), B = h - hd;
        return hd >= (1u << (d - 1)) ? tpi.get(d - 1, B >> d) : tpf.get(d - 1, B >> d);
    };
    // one tile per CTA: every level's twiddles are fetched at once into
    // shared memory (one global-memory latency instead of one per level)
    __shared__ Tw<W> pre2[16], pre3[16];
    const bool pre = !uniform && t < 16;
    if (pre) {
        for (int d = dact + (int)ln.id; d <= t; d += (int)ln.n) {
            pre2[d] = tw2(d);
            pre3[d] = tw3(d);
        }
        __syncthreads();
    }
    Tw<W> wn = !pre && act && t >= dact ? tw2(t) : Tw<W>{};
    Tw<W> wn3 = !pre && act && dact <= t ? tw3(dact) : Tw<W>{};
    // One level's sweep over the element pairs (lo, hi) = (idx, idx + Hw) for
    // idx in [base_idx, base_idx + cnt): rows and columns are one flat index
    // ((pos << wl) | col), so a lane walks it with a constant stride; the
    // padded address of idx + 32 k is that of idx plus 33 k, which makes the
    // stride and (for Hw a multiple of 32) the partner offset constants.
    auto sweep = [&](uint32_t base_idx, uint32_t cnt, uint32_t Hw, auto body) {
        if ((ln.n & 31) == 0 && (Hw & 31) == 0) {
            const uint32_t i0 = base_idx + ln.id;
            W* p = tl.S + i0 + (i0 >> 5);
            const uint32_t off = Hw + (Hw >> 5), step = ln.n + (ln.n >> 5);
            for (uint32_t g = ln.id; g < cnt; g += ln.n, p += step) body(p[0], p[off]);
        } else {
            for (uint32_t g = ln.id; g < cnt; g += ln.n) {
                const uint32_t ia = base_idx + g, ib = ia + Hw;
                body(tl.S[ia + (ia >> 5)], tl.S[ib + (ib >> 5)]);
            }
        }
    };
    // zero_tail: the known tail [h, 2^t) is all zeros (a plain ITFT: every
    // caller but the vector's last chunk).  While the block holding h still
    // has a zero upper half, folding it into the left half is a no-op and
    // splitting it off is a copy (w 0 = 0); the first split makes the tails
    // nonzero.
    bool zt = zero_tail;
    for (int d = t; d >= dlo; --d) {
        const Tw<W> w = pre ? pre2[d] : wn;
        if (!pre && act && d - 1 >= dact) wn = tw2(d - 1);
        if (d >= dact) {
            const uint32_t hd = h & ((1u << d) - 1);
            const uint32_t B = h - hd, H = 1u << (d - 1);
            if (hd >= H && zt) {
                const uint32_t i0 = hd - H;
                sweep((B + i0) << wl, (H - i0) << wl, H << wl, [&](W& lo, W& hi) { hi = lo; });
                zt = false;
            } else if (hd >= H) {
                const uint32_t i0 = hd - H;
                sweep((B + i0) << wl, (H - i0) << wl, H << wl, [&](W& lo, W& hi) {
                    if constexpr (F::kLazy) {  // values stay in [0, 4p)
                        const W m = f.mulw(hi, w);
                        const W x = f.red2(lo) - m + f.p2;
                        lo = x;
                        hi = f.red2(x) - m + f.p2;
                    } else {
                        const W m = f.cmulw(hi, w);
                        const W x = f.csub(f.canon(lo), m);
                        lo = x;
                        hi = f.csub(x, m);
                    }
                });
            } else if (!zt) {
                sweep((B + hd) << wl, (H - hd) << wl, H << wl, [&](W& lo, W& hi) {
                    if constexpr (F::kLazy) lo = f.red2(lo) + f.mulw(hi, w);
                    else lo = f.cadd(lo, f.cmulw(hi, w));
                });
            }
        }
        __syncthreads();
    }
    for (int d = dlo; d <= t; ++d) {
        const Tw<W> w = pre ? pre3[d] : wn3;
        if (!pre && act && d >= dact && d + 1 <= t) wn3 = tw3(d + 1);
        if (d >= dact) {
            const uint32_t hd = h & ((1u << d) - 1);
            const uint32_t B = h - hd, H = 1u << (d - 1);
            if (hd >= H) {
                const uint32_t cnt = (hd - H) << wl;
                const Tw<W> wh = cnt ? f.tw(f.twmul(w, R.inv2)) : w;  // w / 2: one product per element
                sweep(B << wl, cnt, H << wl, [&](W& lo, W& hi) {
                    if constexpr (F::kLazy) {
                        const W l = f.red2(lo), u = f.red2(hi);
                        lo = f.mulw(l + u, R.inv2);
                        hi = f.mulw(l - u + f.p2, wh);
                    } else {
                        const W l = f.canon(lo), u = hi;
                        lo = f.cmulw(f.cadd(l, u), R.inv2);
                        hi = f.cmulw(f.csub(l, u), wh);
                    }
                });
            } else {
                sweep(B << wl, hd << wl, H << wl, [&](W& lo, W& hi) {
                    if constexpr (F::kLazy) lo = f.red2(lo) - f.mulw(hi, w) + f.p2;
                    else lo = f.csub(lo, f.cmulw(hi, w));
                });
            }
        }
        __syncthreads();
    }
}

// Per-column evaluation sum_{i<cnt} S[row0 + i] w^i; w a canonical field word.
// Result per column into out[col] (canonical).  `red` is scratch of
// blockDim.x words.  Ends synced.
//
// The column's next output after an in-tile solve of K known rows (its first
// virtual word, the input of the vector's last chunk): the top-down sweep of
// itft_phases23 leaves, in the slots [K, K + H) with H the lowest set bit of
// K, the residue of the column modulo z^H - omega_K^H (the right child at
// the deepest level that holds K, its coefficients in natural order), and
// nothing writes them afterwards.  So F(omega_K) = sum_{i<H} S[K + i] omega_K^i:
// H terms instead of the K of a Horner pass over the solved coefficients
// (one term, no product at all, when K is odd).
template <class F>
TFT_DEV void colsum_pow(const F& f, const SmemTile<typename F::W>& tl, uint32_t row0, uint32_t cnt,
                        typename F::W wword, typename F::W one, typename F::W* red, typename F::W* out) {
    using W = typename F::W;
    const uint32_t ncols = 1u << tl.wlog;
    if (ncols >= blockDim.x || cnt <= 4) {  // whole columns per thread, Horner over the rows
        const Tw<W> w = f.tw(wword);
        for (uint32_t col = threadIdx.x; col < ncols; col += blockDim.x) {
            W acc = 0;
            for (uint32_t i = cnt; i-- > 0;) acc = f.cadd(f.cmulw(acc, w), f.canon(tl.at(tl.ix(row0 + i, col))));
            out[col] = acc;
        }
        __syncthreads();
        return;
    }
    const uint32_t nparts = blockDim.x >> tl.wlog;
    const uint32_t col = threadIdx.x & (ncols - 1), part = threadIdx.x >> tl.wlog;
    const uint32_t e = (cnt + nparts - 1) / nparts;
    const uint32_t r0 = part * e, r1 = min(cnt, r0 + e);
    const Tw<W> w = f.tw(wword);
    W acc = 0;
    if (r0 < r1) {
        for (uint32_t i = r1; i-- > r0;) acc = f.cadd(f.cmulw(acc, w), f.canon(tl.at(tl.ix(row0 + i, col))));
        acc = f.cmulw(acc, f.tw(pow_w(f, wword, one, r0)));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (part == 0) {
        W s = 0;
        for (uint32_t q = 0; q < nparts; ++q) s = f.cadd(s, red[(q << tl.wlog) | col]);
        out[col] = s;
    }
    __syncthreads();
}

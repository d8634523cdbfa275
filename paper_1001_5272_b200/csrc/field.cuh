// Modular arithmetic for the TFT kernels (sm_100a).
//
// Three word types, chosen per RingConfig by the host:
//   F30 — odd p < 2^30, uint32 words, Harvey lazy butterflies: values live in
//         [0, 4p) between stages and are made canonical at the final store.
//   F32 — odd p < 2^32 (e.g. 3221225473 = 3*2^30+1), uint32 words, canonical
//         [0, p) everywhere (2p does not fit a word, so nothing can be lazy).
//   F62 — odd p < 2^62 (the reference's modulus bound, modring.py:88-89),
//         uint64 words, Harvey lazy butterflies (4p < 2^64).
//
// Twiddles are stored in Montgomery form wM = w*R mod p (R = 2^32 or 2^64)
// together with a companion wMp = wM * (+-p^-1) mod R, so b*w mod p costs
// three integer multiplies and no division (Montgomery reduction with the
// quotient digit m = lo(b*wM) * (+-p^-1) = b*wMp precomputed per twiddle):
//   F30:      m = b*wMp, r = (b*wM + m*p) >> 32          (companion -p^-1)
//   F32/F62:  m = b*wMp, r = hi(b*wM) - hi(m*p) (+p)      (companion +p^-1)
// both exact because the low words cancel.  Results lie in [0, 2p); F32
// folds back to [0, p).
// Reference: the scalar `(u128)a*b % p` of `_kernels.pyx:17-18`.
#pragma once
#include <cstdint>

#define TFT_DEV __device__ __forceinline__

template <typename W>
struct Tw {
    W w;   // Montgomery form
    W wp;  // w * p^-1 mod R
};

struct F30 {
    using W = uint32_t;
    static constexpr bool kLazy = true;
    W p, p2, pinv;  // pinv holds -p^-1 mod 2^32 for this field (REDC sign)

    TFT_DEV W red2(W x) const { return min(x, x - p2); }  // [0,4p) -> [0,2p)
    TFT_DEV W red1(W x) const { return min(x, x - p); }   // [0,2p) -> [0,p)
    TFT_DEV W canon(W x) const { return red1(red2(x)); }
    // b * w for any b < 4p: REDC of T = b*wM with m = b*wMp = lo(T)*(-p^-1):
    // (T + m p) / 2^32 in [0, 2p).  Written as one 64-bit sum so ptxas emits
    // IMAD, IMAD.WIDE and one IMAD.HI with the 64-bit addend (no negations).
    TFT_DEV W mulw(W b, W wM, W wMp) const {
        const uint32_t m = b * wMp;
        const uint64_t t = (uint64_t)b * wM + (uint64_t)m * p;
        return (W)(t >> 32);
    }
    TFT_DEV W mulw(W b, Tw<W> t) const { return mulw(b, t.w, t.wp); }
    // Montgomery product a*b/R for a, b < 2p: [0, 2p)
    TFT_DEV W mont(W a, W b) const {
        const uint64_t ab = (uint64_t)a * b;
        const uint32_t m = (uint32_t)ab * pinv;
        return (W)((ab + (uint64_t)m * p) >> 32);
    }
    TFT_DEV Tw<W> mk(W wM) const { return Tw<W>{wM, wM * pinv}; }
    // Cooley-Tukey (DIT on the remainder tree) butterfly: (a + w b, a - w b).
    // in [0,4p) -> out [0,4p)
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        W a = red2(x);
        W b = mulw(y, t);
        x = a + b;
        y = a - b + p2;
    }
    // Unscaled Gentleman-Sande inverse: (a + b, w^-1 (a - b)).  in [0,2p) -> out [0,2p)
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        W s = red2(x + y);
        W d = x - y + p2;
        x = s;
        y = mulw(d, t);
    }
    TFT_DEV W lazy_in(W x) const { return x; }  // canonical input is a valid lazy value
    // canonical-in/canonical-out helpers (cheap paths of the inverse solver)
    TFT_DEV W cadd(W a, W b) const { return red1(a + b); }
    TFT_DEV W csub(W a, W b) const { return red1(a - b + p); }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return red1(mulw(b, t)); }
};

struct F32 {
    using W = uint32_t;
    static constexpr bool kLazy = false;
    W p, p2, pinv;  // p2 unused

    TFT_DEV W red2(W x) const { return x; }
    TFT_DEV W red1(W x) const { return x; }
    TFT_DEV W canon(W x) const { return x; }
    TFT_DEV W mulw(W b, W wM, W wMp) const {
        W hi = __umulhi(b, wM);
        W m = b * wMp;
        W u = __umulhi(m, p);
        W d = hi - u;
        return hi < u ? d + p : d;
    }
    TFT_DEV W mulw(W b, Tw<W> t) const { return mulw(b, t.w, t.wp); }
    TFT_DEV W mont(W a, W b) const {
        W hi = __umulhi(a, b);
        W m = a * b * pinv;
        W u = __umulhi(m, p);
        W d = hi - u;
        return hi < u ? d + p : d;
    }
    TFT_DEV Tw<W> mk(W wM) const { return Tw<W>{wM, wM * pinv}; }
    TFT_DEV W cadd(W a, W b) const {
        W s = a + b;
        return (s < a || s >= p) ? s - p : s;
    }
    TFT_DEV W csub(W a, W b) const {
        W d = a - b;
        return a < b ? d + p : d;
    }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return mulw(b, t); }
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        W b = mulw(y, t);
        W a = x;
        x = cadd(a, b);
        y = csub(a, b);
    }
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        W s = cadd(x, y);
        W d = csub(x, y);
        x = s;
        y = mulw(d, t);
    }
    TFT_DEV W lazy_in(W x) const { return x; }
};

struct F62 {
    using W = uint64_t;
    static constexpr bool kLazy = true;
    W p, p2, pinv;

    TFT_DEV W red2(W x) const { return min(x, x - p2); }
    TFT_DEV W red1(W x) const { return min(x, x - p); }
    TFT_DEV W canon(W x) const { return red1(red2(x)); }
    TFT_DEV W mulw(W b, W wM, W wMp) const {
        W hi = __umul64hi(b, wM);
        W m = b * wMp;
        return hi - __umul64hi(m, p) + p;
    }
    TFT_DEV W mulw(W b, Tw<W> t) const { return mulw(b, t.w, t.wp); }
    TFT_DEV W mont(W a, W b) const {
        W hi = __umul64hi(a, b);
        W m = a * b * pinv;
        return hi - __umul64hi(m, p) + p;
    }
    TFT_DEV Tw<W> mk(W wM) const { return Tw<W>{wM, wM * pinv}; }
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        W a = red2(x);
        W b = mulw(y, t);
        x = a + b;
        y = a - b + p2;
    }
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        W s = red2(x + y);
        W d = x - y + p2;
        x = s;
        y = mulw(d, t);
    }
    TFT_DEV W lazy_in(W x) const { return x; }
    TFT_DEV W cadd(W a, W b) const { return red1(a + b); }
    TFT_DEV W csub(W a, W b) const { return red1(a - b + p); }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return red1(mulw(b, t)); }
};

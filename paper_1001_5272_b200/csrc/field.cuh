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
// Twiddle multiplication b*w mod p costs three integer multiplies and no
// division, with a per-twiddle companion stored next to w (Tw<W>):
//   F30:      Shoup.  w in normal form, ws = floor(w 2^32 / p);
//             q = hi(b ws), r = b w - q p in [0, 2p) for any 32-bit b.
//             (IMAD.HI + 2 IMAD = 4 FMA-pipe slots on sm_100a; IMAD.HI and
//             IMAD.WIDE issue at half rate, measured, so this beats REDC.)
//   F32/F62:  Montgomery.  wM = w R mod p, companion wM p^-1 mod R;
//             m = b*wMp, r = hi(b wM) - hi(m p) (+p).
// "Field words" are the stored form (normal for F30, Montgomery for F32/F62);
// tw(x) builds a full twiddle from a canonical field word and twmul multiplies
// two twiddles into a field word.  mont(a, b) = a b R^-1 is the
// representation-free product used for data x data (the pointwise product).
// Reference: the scalar `(u128)a*b % p` of `_kernels.pyx:17-18`.
#pragma once
#include <cstdint>
#include <type_traits>

#define TFT_DEV __device__ __forceinline__

template <typename W>
struct Tw {
    W w;   // Montgomery form
    W wp;  // w * p^-1 mod R
};

struct F30 {
    using W = uint32_t;
    static constexpr bool kLazy = true;
    W p, p2, pinv;  // pinv = p^-1 mod 2^32
    W npinv;        // -p^-1 mod 2^32 (REDC)
    W c32, c32s;    // 2^32 mod p as a Shoup twiddle (companion generation)

    TFT_DEV W red2(W x) const { return min(x, x - p2); }  // [0,4p) -> [0,2p)
    TFT_DEV W red1(W x) const { return min(x, x - p); }   // [0,2p) -> [0,p)
    TFT_DEV W canon(W x) const { return red1(red2(x)); }
    // Shoup: b * w for any 32-bit b, result in [0, 2p)
    TFT_DEV W mulw(W b, W w, W ws) const { return b * w - __umulhi(b, ws) * p; }
    TFT_DEV W mulw(W b, Tw<W> t) const { return mulw(b, t.w, t.wp); }
    // Shoup companion of a canonical w: w 2^32 = ws p + r, so ws = -r p^-1 mod 2^32
    TFT_DEV Tw<W> tw(W w) const {
        const W r = red1(mulw(w, c32, c32s));
        return Tw<W>{w, (0u - r) * pinv};
    }
    TFT_DEV W twmul(Tw<W> a, Tw<W> b) const { return red1(mulw(a.w, b)); }
    // b * (constant scale factor, a Shoup pair): [0, 2p)
    TFT_DEV W scale(W b, Tw<W> t) const { return mulw(b, t); }
    // REDC a*b/2^32 for a*b < p 2^32: [0, 2p)
    TFT_DEV W mont(W a, W b) const {
        const uint64_t ab = (uint64_t)a * b;
        const uint32_t m = (uint32_t)ab * npinv;
        return (W)((ab + (uint64_t)m * p) >> 32);
    }
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
    // one output of the butterfly: sel ? a - w b : a + w b (and w = 1)
    TFT_DEV W half(W x, W y, Tw<W> t, bool sel) const {
        const W a = red2(x), b = mulw(y, t);
        return sel ? a - b + p2 : a + b;
    }
    TFT_DEV W half1(W x, W y, bool sel) const {
        const W a = red2(x), b = red2(y);
        return sel ? a - b + p2 : a + b;
    }
    // canonical-in/canonical-out helpers (cheap paths of the inverse solver)
    TFT_DEV W cadd(W a, W b) const { return red1(a + b); }
    TFT_DEV W csub(W a, W b) const { return red1(a - b + p); }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return red1(mulw(b, t)); }
};

// F30 with single-word twiddles: the twiddle is w R mod p (R = 2^32) and its
// companion w R p^-1 mod R is one IMAD from it, so a twiddle costs 4 bytes of
// table instead of 8.  b w = hi(b wR) - hi((b wRp) p) + p in (0, 2p) for any
// 32-bit b: two IMAD.HI + one IMAD, against Shoup's one IMAD.HI + two IMAD.
// Used where twiddles are per-thread (the bottom 5 stages), so table bytes,
// not the integer pipe, are the limit.  Constant scale factors stay Shoup.
struct F30M : F30 {
    TFT_DEV explicit F30M(const F30& f) : F30(f) {}
    TFT_DEV W mulw(W b, Tw<W> t) const { return __umulhi(b, t.w) - __umulhi(b * t.wp, p) + p; }
    TFT_DEV W scale(W b, Tw<W> t) const { return F30::mulw(b, t); }
    // Both outputs straight from hi = hi(y wR) and u = hi((y wRp) p):
    // x = (ra + p) + hi - u, y = (ra + p) - hi + u (ra = red2(x)), the same
    // words as a + b, a - b + 2p with b = hi - u + p.  Written this way
    // ptxas keeps hi - u out of a 64-bit-addend IMAD.HI, whose zeroed and
    // negated operand registers cost two extra FMA-pipe moves per product
    // (tools/cu/engmix.cu: bottom round 6.7 -> 8.8 butterflies/clk/SM).
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W ra = red2(x) + p;
        const W hi = __umulhi(y, t.w);
        const W u = __umulhi(y * t.wp, p);
        x = ra + hi - u;
        y = ra - hi + u;
    }
    // (x - y) w as one REDC of the 64-bit sum d wR + m p, m = d (-wRp):
    // [0, 2p) (engmix: 7.4 -> 7.6)
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        const W s = red2(x + y);
        const W d = x - y + p2;
        x = s;
        const W m = d * (0u - t.wp);
        y = (W)(((uint64_t)d * t.w + (uint64_t)m * p) >> 32);
    }
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
    TFT_DEV Tw<W> tw(W wM) const { return Tw<W>{wM, wM * pinv}; }
    TFT_DEV W twmul(Tw<W> a, Tw<W> b) const { return mont(a.w, b.w); }
    TFT_DEV W scale(W b, Tw<W> t) const { return mulw(b, t); }
    // a + b = a - (p - b): the borrow of the subtraction is the only test
    // (one compare instead of the carry and range tests of a + b)
    TFT_DEV W cadd(W a, W b) const {
        const W nb = p - b;
        const W s = a - nb;
        return a < nb ? s + p : s;
    }
    TFT_DEV W csub(W a, W b) const {
        W d = a - b;
        return a < b ? d + p : d;
    }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return mulw(b, t); }
    // (engmix: forward and inverse rounds +8% over the carry-test cadd)
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W b = mulw(y, t);
        const W a = x;
        x = cadd(a, b);
        y = csub(a, b);
    }
    TFT_DEV W half(W x, W y, Tw<W> t, bool sel) const {
        const W b = mulw(y, t);
        return sel ? csub(x, b) : cadd(x, b);
    }
    TFT_DEV W half1(W x, W y, bool sel) const { return sel ? csub(x, y) : cadd(x, y); }
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        const W a = x, b = y;
        x = cadd(a, b);
        y = mulw(csub(a, b), t);
    }
};

// F32 inside a register round: words are "wide" -- any 32-bit value
// congruent to the residue (2^32 < 2p, so a wide word is the canonical one or
// canonical + p).  The Montgomery product takes any 32-bit multiplicand and
// returns a canonical word, so a butterfly's sum and difference each need only
// the carry (borrow) of one 32-bit add and a predicated +-p: ptxas turns the
// add.cc / addc / setp / @p sequence below into IADD3 (carry predicate) +
// predicated IMAD.IADD.  Per butterfly 5 ALU-pipe + 7 FMA-pipe slots against
// the canonical form's 9 + 6 (cuobjdump, tools/cu/f32wide.cu).  Words are made
// canonical again (narrow) when a round writes its unit back, so tiles in
// shared memory and everything outside the rounds stay canonical.
struct F32W : F32 {
    static constexpr bool kWide = true;
    TFT_DEV explicit F32W(const F32& f) : F32(f) {}
    // a wide, b canonical -> wide
    TFT_DEV W addw(W a, W b) const {
        W d;
        asm("{.reg .u32 m; .reg .pred q;\n\t"
            "add.cc.u32 %0, %1, %2;\n\taddc.u32 m, 0, 0;\n\tsetp.ne.u32 q, m, 0;\n\t"
            "@q sub.u32 %0, %0, %3;}"
            : "=&r"(d) : "r"(a), "r"(b), "r"(p));
        return d;
    }
    TFT_DEV W subw(W a, W b) const {
        W d;
        asm("{.reg .u32 m; .reg .pred q;\n\t"
            "sub.cc.u32 %0, %1, %2;\n\taddc.u32 m, 0, 0;\n\tsetp.eq.u32 q, m, 0;\n\t"
            "@q add.u32 %0, %0, %3;}"
            : "=&r"(d) : "r"(a), "r"(b), "r"(p));
        return d;
    }
    TFT_DEV W narrow(W x) const { return min(x, x - p); }
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W b = mulw(y, t);
        const W a = x;
        x = addw(a, b);
        y = subw(a, b);
    }
    // ycanon: y is known canonical (a tile word, or the product side of the
    // layer below -- a compile-time fact after unrolling, tile.cuh reg_inv)
    TFT_DEV void inv(W& x, W& y, Tw<W> t, bool ycanon = false) const {
        const W a = x, b = ycanon ? y : narrow(y);
        x = addw(a, b);
        y = mulw(subw(a, b), t);
    }
};

// fields whose register rounds hold wide words (narrowed at the write-back)
template <class F, class = void>
struct is_wide : std::false_type {};
template <class F>
struct is_wide<F, std::enable_if_t<F::kWide>> : std::true_type {};

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
    TFT_DEV Tw<W> tw(W wM) const { return Tw<W>{wM, wM * pinv}; }
    TFT_DEV W twmul(Tw<W> a, Tw<W> b) const { return red1(mont(a.w, b.w)); }
    TFT_DEV W scale(W b, Tw<W> t) const { return mulw(b, t); }
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
    TFT_DEV W half(W x, W y, Tw<W> t, bool sel) const {
        const W a = red2(x), b = mulw(y, t);
        return sel ? a - b + p2 : a + b;
    }
    TFT_DEV W half1(W x, W y, bool sel) const {
        const W a = red2(x), b = red2(y);
        return sel ? a - b + p2 : a + b;
    }
    TFT_DEV W cadd(W a, W b) const { return red1(a + b); }
    TFT_DEV W csub(W a, W b) const { return red1(a - b + p); }
    TFT_DEV W cmulw(W b, Tw<W> t) const { return red1(mulw(b, t)); }
};

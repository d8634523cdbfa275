/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's hot path (Harvey & Roche,
 * arXiv 1001.5272; reference package `tftmul` 0.1.0).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the CHECKER (or the timed CPU baseline).
 * The product path (paper_1001_5272_b200/) never links or calls it.
 *
 * Pinned against the reference: tests/golden/ holds vectors produced by the
 * reference itself (tests/golden/make_golden.py imports /root/reference and
 * its compiled _kernels built by oracle/Makefile into oracle/_ref/), and
 * tests/test_oracle.py checks every one of them against this file.
 *
 * Arithmetic: canonical residues in [0,p), p an odd prime < 2^62, products
 * through unsigned __int128 exactly as the reference (`_kernels.pyx:17-18`).
 *
 * Deviation from the reference that does not change any value: butterfly
 * twiddles theta = omega_{2j} are read from a table Z[j] built once per call
 * (the reference regenerates them with a bit-reversed running product,
 * `_kernels.pyx:181-223`).  The traversal follows the paper's recursion
 * (Algorithm 1 / 2), written recursively; depth is
 * bounded by ceil_lg(n) + 1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned long long u64;
typedef unsigned __int128 u128;
typedef long long i64;

static inline u64 mm(u64 a, u64 b, u64 p) { return (u64)(((u128)a * b) % p); }
static inline u64 ad(u64 a, u64 b, u64 p) { u64 s = a + b; return s >= p ? s - p : s; }
static inline u64 sb(u64 a, u64 b, u64 p) { return a >= b ? a - b : a + p - b; }

static int bitlen64(u64 e) { int k = 0; while (e) { e >>= 1; k++; } return k; }
/* ceil_lg (modring.py:49-53) */
static int ceil_lg64(i64 n) { return bitlen64((u64)(n - 1)); }

static u64 pw(u64 a, u64 e, u64 p) {
    u64 r = 1;
    while (e) { if (e & 1) r = mm(r, a, p); a = mm(a, a, p); e >>= 1; }
    return r;
}

/* omega_[k]: the canonical 2^k-th root, omegaK squared K-k times
 * (modring.py:205-220 root_of_level). */
static u64 root_level(int k, u64 p, u64 top, int K) {
    u64 w = top;
    for (int i = 0; i < K - k; i++) w = mm(w, w, p);
    return w;
}

static u64 revbits(u64 s, int k) {
    u64 r = 0;
    for (int i = 0; i < k; i++) { r = (r << 1) | (s & 1); s >>= 1; }
    return r;
}

/* omega_s = omega_[bitlen s]^{rev(s)} (modring.py:223-234). */
u64 orc_omega(u64 s, u64 p, u64 top, int K) {
    if (s == 0) return 1;
    int k = bitlen64(s);
    return pw(root_level(k, p, top, K), revbits(s, k), p);
}

/* Z[j] = omega_{2j} for j < 2^(lg-1).  Z[2^(k-1) + i] = omega_[k+1] * Z[i]
 * because omega_{q+t} = omega_q omega_t whenever 2^k | q and t < 2^k
 * (PAPER.md:425). */
static u64 *twiddle_table(int lg, u64 p, u64 top, int K) {
    i64 sz = lg >= 1 ? ((i64)1 << (lg - 1)) : 1;
    u64 *Z = (u64 *)malloc(sizeof(u64) * (size_t)sz);
    if (!Z) return NULL;
    Z[0] = 1;
    for (int k = 1; k <= lg - 1; k++) {
        u64 w = root_level(k + 1, p, top, K);
        i64 h = (i64)1 << (k - 1);
        for (i64 i = 0; i < h; i++) Z[h + i] = mm(w, Z[i], p);
    }
    return Z;
}

/* omega_s from the table: omega_{2j+1} = -omega_{2j}. */
static inline u64 omega_tab(const u64 *Z, u64 s, u64 p) {
    u64 z = Z[s >> 1];
    return (s & 1) ? (z ? p - z : 0) : z;
}

typedef struct {
    u64 *X; i64 n; u64 p; const u64 *Z; const u64 *Zi;
} walk_t;

/* len(S) = ceil((n-q)/2^r)  (tree.py:20-25, _kernels.pyx:301-302) */
static inline i64 node_len(i64 n, i64 q, int r) {
    return (n - q + ((i64)1 << r) - 1) >> r;
}

/* Odd-tail correction of node S=(q,r) with odd m >= 3
 * (_kernels.pyx:275-298, transforms.py:121-151):
 * v = sum_{i<half} S_{2i+1} omega_half^i, S_{m-1} += sign * v omega_{m-1}. */
static void odd_tail(walk_t *w, i64 q, int r, i64 m, int sign) {
    u64 p = w->p;
    i64 half = (m - 1) >> 1;
    u64 wl = omega_tab(w->Z, (u64)(m - 1), p);
    u64 wh = omega_tab(w->Z, (u64)half, p);
    i64 stride = (i64)1 << r;
    i64 idx = q + (2 * (half - 1) + 1) * stride;
    u64 v = w->X[idx];
    for (i64 i = half - 2; i >= 0; i--) {
        idx -= 2 * stride;
        v = ad(mm(v, wh, p), w->X[idx], p);
    }
    u64 t = mm(v, wl, p);
    i64 last = q + (m - 1) * stride;
    w->X[last] = sign > 0 ? ad(w->X[last], t, p) : sb(w->X[last], t, p);
}

/* Algorithm 1 on node (q,r) (_kernels.pyx:305-335):
 * even subtree, odd-tail correction from the raw odd child, odd subtree,
 * then the node's butterflies (S_2j, S_2j+1) <- (a + theta b, a - theta b),
 * theta = omega_{2j} (_kernels.pyx:181-223). */
static void tft_node(walk_t *w, i64 q, int r) {
    i64 m = node_len(w->n, q, r);
    if (m <= 1) return;
    tft_node(w, q, r + 1);
    if (m & 1) odd_tail(w, q, r, m, +1);
    tft_node(w, q + ((i64)1 << r), r + 1);
    u64 p = w->p;
    i64 stride = (i64)1 << r;
    for (i64 j = 0; j < (m >> 1); j++) {
        i64 lo = q + j * 2 * stride, hi = lo + stride;
        u64 a = w->X[lo], b = mm(w->X[hi], w->Z[j], p);
        w->X[lo] = ad(a, b, p);
        w->X[hi] = sb(a, b, p);
    }
}

/* Algorithm 2 on node (q,r) (_kernels.pyx:338-363): the
 * exact mirror — inverse butterflies ((a+b)/2, theta^-1 (a-b)/2), the odd
 * subtree, removal of the odd-tail correction (now computable from the
 * restored odd child), then the even subtree. */
static void itft_node(walk_t *w, i64 q, int r, u64 inv2) {
    i64 m = node_len(w->n, q, r);
    if (m <= 1) return;
    u64 p = w->p;
    i64 stride = (i64)1 << r;
    for (i64 j = 0; j < (m >> 1); j++) {
        i64 lo = q + j * 2 * stride, hi = lo + stride;
        u64 a = w->X[lo], b = w->X[hi];
        u64 s = mm(ad(a, b, p), inv2, p);
        u64 d = mm(sb(a, b, p), inv2, p);
        if (j) d = mm(d, w->Zi[j], p);
        w->X[lo] = s;
        w->X[hi] = d;
    }
    itft_node(w, q + stride, r + 1, inv2);
    if (m & 1) odd_tail(w, q, r, m, -1);
    itft_node(w, q, r + 1, inv2);
}

/* transforms.tft (transforms.py:208-224) without the Python-side checks.
 * Returns 0, or -1 on bad arguments / allocation failure. */
int orc_tft(u64 *x, i64 n, u64 p, u64 top, int K) {
    if (n <= 0 || ceil_lg64(n) > K) return -1;
    if (n == 1) return 0;
    u64 *Z = twiddle_table(ceil_lg64(n), p, top, K);
    if (!Z) return -1;
    walk_t w = {x, n, p, Z, NULL};
    tft_node(&w, 0, 0);
    free(Z);
    return 0;
}

/* transforms.itft (transforms.py:227-237). */
int orc_itft(u64 *x, i64 n, u64 p, u64 top, int K) {
    if (n <= 0 || ceil_lg64(n) > K) return -1;
    if (n == 1) return 0;
    int lg = ceil_lg64(n);
    u64 *Z = twiddle_table(lg, p, top, K);
    /* inverse twiddles theta^-1: the same table built from omegaK^-1 (the
     * reference advances theta^-1 from the inverse base root,
     * _kernels.pyx:116-123, 226-272) */
    u64 *Zi = twiddle_table(lg, p, pw(top, p - 2, p), K);
    if (!Z || !Zi) { free(Z); free(Zi); return -1; }
    walk_t w = {x, n, p, Z, Zi};
    itft_node(&w, 0, 0, (p + 1) >> 1);
    free(Z);
    free(Zi);
    return 0;
}

static void fold_twist(const u64 *src, i64 ls, u64 *X, i64 base, i64 L, u64 wq, u64 p) {
    /* X[base + (i mod L)] += omega_q^i src[i]  (polymul.py:55-88,
     * _kernels.pyx:366-398) */
    u64 pwq = 1;
    i64 idx = base;
    for (i64 i = 0; i < ls; i++) {
        X[idx] = ad(X[idx], mm(src[i], pwq, p), p);
        pwq = mm(pwq, wq, p);
        if (++idx == base + L) idx = base;
    }
}

static u64 horner(const u64 *poly, i64 nc, u64 pt, u64 p) {
    /* polymul.horner_eval (polymul.py:39-52) */
    u64 acc = poly[nc - 1];
    for (i64 i = nc - 2; i >= 0; i--) acc = ad(mm(acc, pt, p), poly[i], p);
    return acc;
}

/* Algorithm 3 (polymul.py:91-141; _kernels.pyx:433-480):
 * for each block (q, L) of the greedy schedule, twisted folds of A and B into
 * X[q:q+L) and X[q+L:q+2L), two power-of-two transforms, a pointwise product;
 * the last slot from two Horner evaluations; one ITFT over X[0:r). */
int orc_multiply(const u64 *a, i64 la, const u64 *b, i64 lb, u64 *x,
                 u64 p, u64 top, int K) {
    if (la <= 0 || lb <= 0) return -1;
    i64 r = la + lb - 1;
    if (ceil_lg64(r) > K) return -1;
    i64 q = 0;
    /* greedy power-of-two cover of [0, r-1) (polymul.py:25-36) */
    while (q < r - 1) {
        int ell = bitlen64((u64)(r - q)) - 2;
        i64 L = (i64)1 << ell;
        memset(x + q, 0, sizeof(u64) * (size_t)(2 * L));
        u64 wq = orc_omega((u64)q, p, top, K);
        fold_twist(a, la, x, q, L, wq, p);
        if (orc_tft(x + q, L, p, top, K)) return -1;
        fold_twist(b, lb, x, q + L, L, wq, p);
        if (orc_tft(x + q + L, L, p, top, K)) return -1;
        for (i64 i = q; i < q + L; i++) x[i] = mm(x[i], x[i + L], p);
        q += L;
    }
    u64 wl = orc_omega((u64)(r - 1), p, top, K);
    x[r - 1] = mm(horner(a, la, wl, p), horner(b, lb, wl, p), p);
    return orc_itft(x, r, p, top, K);
}

/* oracle.naive_dft (oracle.py:46-63): evaluate F at omega_0..omega_{n-1}. */
int orc_naive_dft(const u64 *f, i64 n, u64 *out, u64 p, u64 top, int K) {
    if (n <= 0 || ceil_lg64(n) > K) return -1;
    for (i64 s = 0; s < n; s++) {
        u64 ws = orc_omega((u64)s, p, top, K), acc = 0, wp = 1;
        for (i64 i = 0; i < n; i++) { acc = ad(acc, mm(f[i], wp, p), p); wp = mm(wp, ws, p); }
        out[s] = acc;
    }
    return 0;
}

/* oracle.schoolbook_mul (oracle.py:66-76). */
int orc_schoolbook(const u64 *a, i64 la, const u64 *b, i64 lb, u64 *out, u64 p) {
    if (la <= 0 || lb <= 0) return -1;
    memset(out, 0, sizeof(u64) * (size_t)(la + lb - 1));
    for (i64 i = 0; i < la; i++)
        for (i64 j = 0; j < lb; j++) out[i + j] = ad(out[i + j], mm(a[i], b[j], p), p);
    return 0;
}

/* Batched helpers for the CPU baseline / large parity sweeps: transform
 * `count` vectors laid out back to back, lengths lens[i]. */
int orc_tft_batch(u64 *x, const i64 *lens, i64 count, u64 p, u64 top, int K) {
    i64 off = 0;
    for (i64 i = 0; i < count; i++) { if (orc_tft(x + off, lens[i], p, top, K)) return -1; off += lens[i]; }
    return 0;
}

int orc_itft_batch(u64 *x, const i64 *lens, i64 count, u64 p, u64 top, int K) {
    i64 off = 0;
    for (i64 i = 0; i < count; i++) { if (orc_itft(x + off, lens[i], p, top, K)) return -1; off += lens[i]; }
    return 0;
}

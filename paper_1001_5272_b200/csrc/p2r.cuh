// Lengths just above a power of two: n = 2^k + r, 1 <= r <= kP2RMax.
//
// The network's top stage pairs (j, j + 2^k) with twiddle 1, and only the
// first r of those pairs have a nonzero upper input.  So (DIT on the
// remainder tree: F mod X^(2^k) - 1 and F mod X^(2^k) + 1)
//   * outputs [0, 2^k) are the plain 2^k transform of u_j = x_j + x_{j+2^k}
//     (the fold only touches j < r), and
//   * output 2^k + s is F(rho_s), rho_s = omega_{2^k + s}: a dot product
//     of the n inputs with the powers of rho_s.
// Inverse: the 2^k inverse gives u; with z_t = x_{2^k+t} (t < r) and
// rho_s^(2^k) = -1,
//   y_{2^k+s} = sum_j u_j rho_s^j - 2 sum_{t<r} z_t rho_s^t,
// an r x r Vandermonde system (V[s][t] = rho_s^t, inverted on the host) for
// z; then x_t = u_t - z_t.  The cost over 2^k is one read of the vector with
// r products per word, instead of a two-pass plan whose column networks are
// twice as tall as the data (the time jump the TFT exists to avoid).
#pragma once
#include "cluster.cuh"

constexpr int kP2RMaxDev = 4;  // = tftb::kP2RMax

template <class F>
struct P2RConsts {
    Tw<typename F::W> vinv[kP2RMaxDev][kP2RMaxDev];  // V^-1 as field twiddles
};

// One kernel per direction: the sums S_s = sum_{j < m} x_j rho_s^j (s < r)
// of every vector, then -- in the last block to finish that vector (an
// atomic ticket) -- the fix-up.  The vector is walked in rows of 1024 words
// (thread t owns words 4t..4t+3 of a row: an inner Horner in rho_s); block b
// takes rows b, b + nb, ... in descending order (an outer Horner in
// rho_s^(1024 nb)); the factor rho_s^(1024 b) rho_s^(4t) comes last.  All
// powers are host-built (tab, per s: rho, rho^(1024 nb), rho^(4t) for
// t < 256, rho^(1024 b) for b < nb).
//   forward (INV = false): x_s += x_{2^k+s}, then x_{2^k+s} <- S_s;
//   inverse (INV = true, S from the inverted prefix u):
//     z = V^-1 ((S - y) / 2); x_{2^k+t} = z_t, x_t = u_t - z_t.
// grid (nb, vectors), 256 threads; part: nb x kP2RMaxDev words per vector;
// ticket: one zeroed counter per vector (left zeroed again).
template <class F, bool INV>
__global__ void __launch_bounds__(256) k_p2r(LaunchArgs<F> a, int k, int r, int64_t len, typename F::W* part,
                                             unsigned* ticket, const Tw<typename F::W>* tab, P2RConsts<F> c) {
    using W = typename F::W;
    constexpr int RW = 1024, U = 4;  // words per row, rows in flight
    __shared__ W red[kP2RMaxDev][256];
    __shared__ bool last;
    const F f = a.f;
    const int64_t v = a.vbase + blockIdx.y, vrel = v - a.vbase;
    const int64_t o = a.xd.o(v);
    W* x = a.x + o;
    const int64_t m = min(len, a.xd.n(v));
    const uint32_t nb = gridDim.x, b = blockIdx.x, t = threadIdx.x;
    const int64_t rows = (m + RW - 1) / RW;
    const uint32_t per_s = 2 + 256 + nb;
    Tw<W> rho[kP2RMaxDev], step[kP2RMaxDev];
#pragma unroll
    for (int s = 0; s < kP2RMaxDev; ++s) {
        if (s >= r) continue;
        rho[s] = tab[s * per_s];
        step[s] = tab[s * per_s + 1];
    }
    W acc[kP2RMaxDev] = {};
    Tw<W> rho2[kP2RMaxDev], rho3[kP2RMaxDev];
#pragma unroll
    for (int s = 0; s < kP2RMaxDev; ++s) {
        if (s >= r) continue;
        rho2[s] = f.tw(f.twmul(rho[s], rho[s]));
        rho3[s] = f.tw(f.twmul(rho2[s], rho[s]));
    }
    // one row's four words: e0 + e1 rho + e2 rho^2 + e3 rho^3 (independent
    // products), then the outer Horner step
    auto fold = [&](W e0, W e1, W e2, W e3) {
#pragma unroll
        for (int s = 0; s < kP2RMaxDev; ++s) {
            if (s >= r) continue;
            const W in = f.cadd(f.cadd(e0, f.cmulw(e1, rho[s])), f.cadd(f.cmulw(e2, rho2[s]), f.cmulw(e3, rho3[s])));
            acc[s] = f.cadd(f.cmulw(acc[s], step[s]), in);
        }
    };
    // this block's rows are b + j nb; walk them top down
    if (rows > (int64_t)b) {
        int64_t j = (rows - 1 - b) / nb;
        const int64_t top = b + j * (int64_t)nb;
        if ((top + 1) * RW > m) {  // the partial last row of the vector
            const int64_t base = top * RW + 4 * t;
            W e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) e[q] = base + q < m ? __ldcg(x + base + q) : W(0);
            fold(e[0], e[1], e[2], e[3]);
            --j;
        }
        // full rows, U per step, the next step's loads issued before the folds
        const W* rp = x + (b + j * (int64_t)nb) * RW + 4 * t;  // row b + j nb, word 4t
        const int64_t dn = (int64_t)nb * RW;
        if (((uintptr_t)x & 15) == 0 && sizeof(W) == 4) {
            using V = typename Vec16<W>::T;
            V cur[U], nxt[U];
            auto ld = [&](int64_t jj, const W* ptr, V* e) {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (jj - u >= 0) e[u] = __ldcg(reinterpret_cast<const V*>(ptr - u * dn));
            };
            ld(j, rp, cur);
            for (; j >= 0; j -= U, rp -= U * dn) {
                if (j - U >= 0) ld(j - U, rp - U * dn, nxt);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (j - u >= 0)
                        fold(Vec16<W>::get(cur[u], 0), Vec16<W>::get(cur[u], 1), Vec16<W>::get(cur[u], 2),
                             Vec16<W>::get(cur[u], 3));
#pragma unroll
                for (int u = 0; u < U; ++u) cur[u] = nxt[u];
            }
        } else {
            for (; j >= 0; --j, rp -= dn) fold(__ldcg(rp), __ldcg(rp + 1), __ldcg(rp + 2), __ldcg(rp + 3));
        }
    }
#pragma unroll
    for (int s = 0; s < kP2RMaxDev; ++s) {
        if (s >= r) continue;
        red[s][t] = f.cmulw(f.cmulw(acc[s], tab[s * per_s + 2 + t]), tab[s * per_s + 2 + 256 + b]);
    }
    __syncthreads();
    for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
        if (t < w)
            for (int s = 0; s < r; ++s) red[s][t] = f.cadd(red[s][t], red[s][t + w]);
        __syncthreads();
    }
    W* pv = part + (size_t)vrel * nb * kP2RMaxDev;
    if (t < (uint32_t)r) pv[b * kP2RMaxDev + t] = red[t][0];
    // the last block of this vector sums the partials and applies the fix
    __threadfence();
    __syncthreads();
    if (t == 0) last = atomicAdd(ticket + vrel, 1u) == nb - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int s = 0; s < r; ++s) {
        W sum = 0;
        for (uint32_t q = t; q < nb; q += blockDim.x) sum = f.cadd(sum, __ldcg(pv + q * kP2RMaxDev + s));
        red[s][t] = sum;
    }
    __syncthreads();
    for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
        if (t < w)
            for (int s = 0; s < r; ++s) red[s][t] = f.cadd(red[s][t], red[s][t + w]);
        __syncthreads();
    }
    if (t) return;
    ticket[vrel] = 0;
    const int64_t H = 1ll << k;
    if constexpr (!INV) {
        for (int s = 0; s < r; ++s) {
            x[s] = f.cadd(x[s], x[H + s]);
            x[H + s] = red[s][0];
        }
    } else {
        W rhs[kP2RMaxDev];
        for (int s = 0; s < r; ++s) {
            const W y = f.canon(load_pre(a, o + H + s, x[H + s]));
            rhs[s] = f.cmulw(f.csub(red[s][0], y), a.R.inv2);
        }
        for (int q = 0; q < r; ++q) {
            W z = 0;
            for (int s = 0; s < r; ++s) z = f.cadd(z, f.cmulw(rhs[s], c.vinv[q][s]));
            x[H + q] = z;
            x[q] = f.csub(x[q], z);
        }
    }
}

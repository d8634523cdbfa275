// Host side of libtftb200.so: ring tables, planning, launches and the C ABI
// declared in include/tftb200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tftb200.h"
#include "host.h"
#include "kernels.cuh"
#include "tally.h"

namespace tftb {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
unsigned long long* g_tail_timing = nullptr;
thread_local int64_t g_aux_cur = 0, g_aux_peak = 0;
thread_local int64_t g_stage_cur = 0, g_stage_peak = 0;

template <typename W>
struct TableBuilder {
    uint64_t p;
    int bits;
    W pinv;
    bool shoup;   // F30: {w, floor(w 2^32 / p)}; else Montgomery {wR, wR p^-1}
    uint64_t to_m(uint64_t w) const { return (uint64_t)(((u128)w << bits) % p); }
    Tw<W> tw(uint64_t w) const {
        if (shoup) return Tw<W>{(W)w, (W)(((u128)w << 32) / p)};
        W wm = (W)to_m(w);
        return Tw<W>{wm, (W)(wm * pinv)};
    }
};

template <typename W>
int build_tables(RingHost* rh, RingDev<W>* out) {
    const uint64_t p = rh->p;
    TableBuilder<W> tb{p, (int)(8 * sizeof(W)), inv_word<W>((W)p), rh->kind == 0};
    // omega_[k] = top^(2^(K-k))
    std::vector<uint64_t> lvl(rh->K + 1), ilvl(rh->K + 1);
    uint64_t itop = powmod(rh->top, p - 2, p);
    {
        uint64_t w = rh->top, iw = itop;
        for (int k = rh->K; k >= 0; --k) {
            lvl[k] = w;
            ilvl[k] = iw;
            w = mulmod(w, w, p);
            iw = mulmod(iw, iw, p);
        }
    }
    const int zb = rh->zb, zh = rh->zh;
    const size_t nz = (size_t)1 << zb, nh = (size_t)1 << zh;
    // Z[2^(k-1) + i] = omega_[k+1] * Z[i]  (product rule)
    auto build = [&](const std::vector<uint64_t>& L, std::vector<uint64_t>& Z, int shift) {
        // Z[i] = omega_{2 i 2^shift}; Z[2^(k-1)+i] = omega_[k+1+shift] Z[i]
        Z[0] = 1;
        for (size_t h = 1, k = 1; h < Z.size(); h <<= 1, ++k)
            for (size_t i = 0; i < h; i++) Z[h + i] = mulmod(L[k + 1 + shift], Z[i], p);
    };
    std::vector<uint64_t> zf(nz), zi(nz), zfh(nh), zih(nh);
    build(lvl, zf, 0);
    build(ilvl, zi, 0);
    build(lvl, zfh, zb);
    build(ilvl, zih, zb);
    std::vector<Tw<W>> host;
    host.reserve(2 * nz + 2 * nh + 64 + 8 * 72);
    for (auto v : zf) host.push_back(tb.tw(v));
    for (auto v : zi) host.push_back(tb.tw(v));
    for (auto v : zfh) host.push_back(tb.tw(v));
    for (auto v : zih) host.push_back(tb.tw(v));
    uint64_t inv2 = (p + 1) >> 1, ip = 1;
    for (int k = 0; k < 64; k++) {
        host.push_back(tb.tw(ip));
        ip = mulmod(ip, inv2, p);
    }
    // small-column solvers: V_m^-1 for the first m points omega_0..omega_{m-1}
    // (V_m[s][i] = omega_s^i) and the next-point row omega_m^i, m = 1..8
    auto omega_s = [&](uint64_t sidx) -> uint64_t {
        if (sidx == 0) return 1;
        int k = 64 - __builtin_clzll(sidx);
        uint64_t r = 0, t = sidx;
        for (int i = 0; i < k; i++) { r = (r << 1) | (t & 1); t >>= 1; }
        return k <= rh->K ? powmod(lvl[k], r, p) : 0;
    };
    // three variants: plain; every column scaled by 2^-CL (all
    // rows come from unscaled chunk inverses); all but the last column scaled
    // (the last row comes from the solved partial chunk, already exact)
    const int CLs = sizeof(W) == 4 ? 14 : 13;
    const uint64_t sc = powmod((p + 1) >> 1, CLs, p);
    std::vector<Tw<W>> blocks[3];
    for (int m = 1; m <= 8; m++) {
        std::vector<uint64_t> A(m * 2 * m, 0);
        for (int r = 0; r < m; r++) {
            uint64_t w = omega_s(r), pw = 1;
            for (int c = 0; c < m; c++) { A[r * 2 * m + c] = pw; pw = mulmod(pw, w, p); }
            A[r * 2 * m + m + r] = 1;
        }
        bool ok = (int)rh->K >= (m > 1 ? 64 - __builtin_clzll((uint64_t)(m - 1)) : 0);
        for (int c = 0; c < m && ok; c++) {  // Gauss-Jordan mod p
            int piv = -1;
            for (int r = c; r < m; r++) if (A[r * 2 * m + c]) { piv = r; break; }
            if (piv < 0) { ok = false; break; }
            for (int k = 0; k < 2 * m; k++) std::swap(A[c * 2 * m + k], A[piv * 2 * m + k]);
            uint64_t inv = powmod(A[c * 2 * m + c], p - 2, p);
            for (int k = 0; k < 2 * m; k++) A[c * 2 * m + k] = mulmod(A[c * 2 * m + k], inv, p);
            for (int r = 0; r < m; r++) {
                if (r == c || !A[r * 2 * m + c]) continue;
                uint64_t f = A[r * 2 * m + c];
                for (int k = 0; k < 2 * m; k++)
                    A[r * 2 * m + k] = (A[r * 2 * m + k] + p - mulmod(f, A[c * 2 * m + k], p)) % p;
            }
        }
        for (int var = 0; var < 3; var++) {
            for (int r = 0; r < 8; r++)
                for (int c = 0; c < 8; c++) {
                    uint64_t e = ok && r < m && c < m ? A[r * 2 * m + m + c] : 0;
                    if (var == 1 || (var == 2 && c < m - 1)) e = mulmod(e, sc, p);
                    blocks[var].push_back(tb.tw(e));
                }
            uint64_t wn = omega_s(m), pw = 1;
            for (int c = 0; c < 8; c++) {
                blocks[var].push_back(tb.tw(ok && c < m ? pw : 0));
                pw = mulmod(pw, wn, p);
            }
        }
    }
    for (int var = 0; var < 3; var++) host.insert(host.end(), blocks[var].begin(), blocks[var].end());
    // the same 3 x 8 x 72 entries as raw Montgomery words (w R mod p), packed
    // two per Tw slot, for the REDC dot products of the column solves
    {
        std::vector<W> raw;
        for (int var = 0; var < 3; var++)
            for (auto& t : blocks[var]) {
                uint64_t w = tb.shoup ? (uint64_t)t.w : 0;  // normal form for Shoup fields
                raw.push_back(tb.shoup ? (W)tb.to_m(w) : t.w);
            }
        for (size_t i = 0; i < raw.size(); i += 2) host.push_back(Tw<W>{raw[i], raw[i + 1]});
    }
    // single-word twiddle tables (w R mod p) for the bottom rounds of u32
    // rings (cluster.cuh TwDirectM/TwBigM): Zf, Zi, Zfh, Zih
    const size_t mword_off = host.size();
    constexpr bool words = sizeof(W) == 4;
    if (words) {
        std::vector<W> mw;
        for (auto* z : {&zf, &zi, &zfh, &zih})
            for (auto v : *z) mw.push_back((W)tb.to_m(v));
        if (mw.size() & 1) mw.push_back(0);
        for (size_t i = 0; i < mw.size(); i += 2) host.push_back(Tw<W>{mw[i], mw[i + 1]});
    }
    size_t tw_bytes = host.size() * sizeof(Tw<W>);
    CK(cudaMalloc(&rh->dmem, tw_bytes));
    CK(cudaMemcpy(rh->dmem, host.data(), tw_bytes, cudaMemcpyHostToDevice));
    Tw<W>* d = (Tw<W>*)rh->dmem;
    out->Zf = d;
    out->Zi = d + nz;
    out->Zfh = d + 2 * nz;
    out->Zih = d + 2 * nz + nh;
    out->ipow2 = d + 2 * nz + 2 * nh;
    out->vinv = d + 2 * nz + 2 * nh + 64;
    out->vinvS = out->vinv + 8 * 72;
    out->vinvT = out->vinv + 16 * 72;
    out->vinvM = reinterpret_cast<const W*>(out->vinv + 24 * 72);
    if (words) {
        const W* mw = reinterpret_cast<const W*>(d + mword_off);
        out->ZfM = mw;
        out->ZiM = mw + nz;
        out->ZfhM = mw + 2 * nz;
        out->ZihM = mw + 2 * nz + nh;
    } else {
        out->ZfM = out->ZiM = out->ZfhM = out->ZihM = nullptr;
    }
    uint64_t R1 = tb.to_m(1);
    out->r2w = (W)tb.to_m(R1);  // R^2 mod p
    out->inv2 = tb.tw(inv2);
    out->oneW = tb.shoup ? (W)1 : (W)R1;
    out->zb = zb;
    out->zh = zh;
    return 0;
}

// F32W's difference (field.cuh) reads the carry flag sub.cc leaves behind with
// an addc, which relies on how this toolchain encodes a borrow.  Checked once
// per process on the device, so a different convention fails loudly at ring
// creation instead of giving wrong residues.
__global__ void k_f32w_probe(F32 f0, unsigned* bad) {
    const F32W f(f0);
    const uint32_t p = f.p;
    const uint32_t as[] = {0u, 1u, p - 1, p, p + 1, 0xFFFFFFFFu, 0x80000000u, 1073741823u, 1073741824u};
    const uint32_t bs[] = {0u, 1u, p - 1, p >> 1, 1073741824u, 2147483648u};
    unsigned n = 0;
    for (uint32_t a : as)
        for (uint32_t b : bs) {
            const uint64_t ar = a % p;
            if (f.addw(a, b) % p != (ar + b) % p) ++n;
            if (f.subw(a, b) % p != (ar + p - b) % p) ++n;
        }
    *bad = n;
}
int f32w_probe(uint64_t p) {
    static std::map<std::pair<int, uint64_t>, bool> done;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (done[{dev, p}]) return 0;
    F32 f{};
    f.p = (uint32_t)p;
    f.pinv = inv_word<uint32_t>((uint32_t)p);
    unsigned* d = nullptr;
    unsigned h = 1;
    CK(cudaMalloc(&d, sizeof(unsigned)));
    k_f32w_probe<<<1, 1>>>(f, d);
    cudaError_t e = cudaMemcpy(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(std::string("F32W probe: ") + cudaGetErrorString(e));
    if (h) return fail("F32W carry-flag probe failed: rebuild field.cuh's subw for this toolchain");
    done[{dev, p}] = true;
    return 0;
}

std::mutex g_ring_mu;
std::map<std::tuple<uint64_t, uint64_t, int, int>, std::unique_ptr<RingHost>> g_rings;

int get_ring(uint64_t p, uint64_t top, int K, RingHost** out) {
    if (p < 3 || !(p & 1) || p >= (1ull << 62)) return fail("modulus must be an odd prime below 2^62");
    if (K < 0 || K > 62 || top == 0 || top >= p) return fail("bad root / K");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ring_mu);
    static std::map<int, bool> pool_tuned;
    if (!pool_tuned[dev]) {
        // keep freed stream-ordered allocations cached: re-mapping GBs of
        // scratch costs ~40 ms per call otherwise (measured)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_tuned[dev] = true;
    }
    auto key = std::make_tuple(p, top, K, dev);
    auto it = g_rings.find(key);
    if (it != g_rings.end()) {
        *out = it->second.get();
        return 0;
    }
    auto rh = std::make_unique<RingHost>();
    rh->p = p;
    rh->top = top;
    rh->K = K;
    rh->wbytes = p < (1ull << 32) ? 4 : 8;
    rh->kind = p < (1ull << 30) ? 0 : (p < (1ull << 32) ? 1 : 2);
    int km1 = K > 0 ? K - 1 : 0;
    static const int zb_max = getenv("TFTB_ZB") ? atoi(getenv("TFTB_ZB")) : 16;  // A/B knob
    rh->zb = std::min(km1, zb_max);
    rh->zh = std::min(km1 - rh->zb, 16);
    int rc = rh->wbytes == 4 ? build_tables<uint32_t>(rh.get(), &rh->r32)
                             : build_tables<uint64_t>(rh.get(), &rh->r64);
    if (rc) return rc;
    if (rh->kind == 1 && (rc = f32w_probe(p))) return rc;
    *out = rh.get();
    g_rings[key] = std::move(rh);
    return 0;
}

// ------------------------------------------------------------ host contexts
// The host-pointer entry points run on a non-blocking stream leased from a
// per-device pool: one per concurrently active caller thread.  Calls on
// distinct buffers from different threads therefore overlap on the device,
// as the reference's nogil kernels do on CPU cores (_kernels.pyx:419,428,453),
// and nothing runs on the legacy default stream.  Device staging comes from
// the stream-ordered pool (cached, get_ring sets its release threshold).
struct HostCtx {
    int dev;
    cudaStream_t st;
    // pinned staging for pageable caller buffers (grow-only, up to
    // kPinMax): DMA from page-locked memory instead of the driver's shared
    // bounce buffer, which serialises concurrent callers
    void* pin = nullptr;
    size_t pin_cap = 0;
    int pin_reserve(size_t bytes) {
        if (bytes <= pin_cap) return 0;
        if (pin) cudaFreeHost(pin);
        pin = nullptr;
        pin_cap = 0;
        size_t cap = std::max<size_t>(bytes, 1 << 20);
        cap = (cap + (1 << 20) - 1) & ~(size_t)((1 << 20) - 1);
        CK(cudaHostAlloc(&pin, cap, cudaHostAllocDefault));
        pin_cap = cap;
        return 0;
    }
};
constexpr size_t kPinMax = 64u << 20;

inline bool host_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
std::mutex g_ctx_mu;
std::map<int, std::vector<HostCtx*>> g_ctx_free;

struct CtxLease {
    HostCtx* c = nullptr;
    int acquire() {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lk(g_ctx_mu);
            auto& v = g_ctx_free[dev];
            if (!v.empty()) {
                c = v.back();
                v.pop_back();
                return 0;
            }
        }
        std::unique_ptr<HostCtx> n(new HostCtx{dev, nullptr});
        CK(cudaStreamCreateWithFlags(&n->st, cudaStreamNonBlocking));
        c = n.release();
        return 0;
    }
    cudaStream_t stream() const { return c->st; }
    ~CtxLease() {
        if (!c) return;
        // nothing of this call may still touch the caller's buffers (error
        // paths included) once it returns
        cudaStreamSynchronize(c->st);
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        g_ctx_free[c->dev].push_back(c);
    }
};

// model op counts of the device algorithm
// Host uint64 words <-> device words of a u32 ring through a bounded u64
// staging buffer (kStageWords): device memory is the ring words (4 B/word)
// plus the staging, not 12 B/word.  The pieces are stream-ordered on st, so
// the staging is reused safely; PCIe dominates, the conversion kernels are
// small.  u64 rings copy straight into their words.
constexpr int64_t kStageWords = 1 << 22;  // 32 MB

template <typename W>
int upload_words(W* d, const uint64_t* h, int64_t n, uint64_t* stage, cudaStream_t st) {
    if constexpr (sizeof(W) == 8) {
        CK(cudaMemcpyAsync(d, h, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    } else {
        for (int64_t i = 0; i < n; i += kStageWords) {
            const int64_t m = std::min(kStageWords, n - i);
            CK(cudaMemcpyAsync(stage, h + i, (size_t)m * 8, cudaMemcpyHostToDevice, st));
            const int nb = (int)std::min<int64_t>((m + 255) / 256, 148 * 16);
            k_u64_to_w<W><<<nb, 256, 0, st>>>(stage, d + i, m);
            g_launches++;
        }
    }
    return 0;
}

template <typename W>
int download_words(uint64_t* h, const W* d, int64_t n, uint64_t* stage, cudaStream_t st) {
    if constexpr (sizeof(W) == 8) {
        CK(cudaMemcpyAsync(h, d, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    } else {
        for (int64_t i = 0; i < n; i += kStageWords) {
            const int64_t m = std::min(kStageWords, n - i);
            const int nb = (int)std::min<int64_t>((m + 255) / 256, 148 * 16);
            k_w_to_u64<W><<<nb, 256, 0, st>>>(d + i, stage, m);
            g_launches++;
            CK(cudaMemcpyAsync(h + i, stage, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
        }
    }
    return 0;
}

int host_tft_common(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, bool inverse, int64_t* mults,
                    int64_t* adds) {
    if (n <= 0) return fail("cannot transform an empty buffer");
    if (K < 62 && n > (1ll << K)) return fail("length exceeds 2^K");
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    CtxLease lease;
    if (lease.acquire()) return -1;
    cudaStream_t st = lease.stream();
    const size_t wb = rh->wbytes;
    // device: the n ring words, plus (u32 rings) a bounded u64 staging
    const int64_t sw = wb == 4 ? std::min(n, kStageWords) : 0;
    const size_t wbytes = ((size_t)n * wb + 255) & ~(size_t)255;
    Scratch buf;
    if (buf.get(wbytes + (size_t)sw * 8, st)) return -1;
    void* dw = buf.p;
    uint64_t* stage = (uint64_t*)((char*)buf.p + wbytes);
    uint64_t* hx = x;
    if ((size_t)n * 8 <= kPinMax && !host_pinned(x)) {
        if (lease.c->pin_reserve((size_t)n * 8)) return -1;
        hx = (uint64_t*)lease.c->pin;
        memcpy(hx, x, (size_t)n * 8);
    }
    int rc = 0;
    if (wb == 4) {
        if (upload_words((uint32_t*)dw, hx, n, stage, st)) return -1;
        rc = rh->kind == 0 ? dispatch_tft<F30>(rh, dw, 1, n, n, nullptr, nullptr, inverse, st)
                           : dispatch_tft<F32>(rh, dw, 1, n, n, nullptr, nullptr, inverse, st);
        if (rc) return rc;
        if (download_words(hx, (const uint32_t*)dw, n, stage, st)) return -1;
    } else {
        if (upload_words((uint64_t*)dw, hx, n, stage, st)) return -1;
        rc = dispatch_tft<F62>(rh, dw, 1, n, n, nullptr, nullptr, inverse, st);
        if (rc) return rc;
        if (download_words(hx, (const uint64_t*)dw, n, stage, st)) return -1;
    }
    CK(cudaStreamSynchronize(st));
    if (hx != x) memcpy(x, hx, (size_t)n * 8);
    tally_transform(n, p, K, inverse, mults, adds);
    return 0;
}

}  // namespace tftb

using namespace tftb;


// ====================================================================== C ABI
extern "C" {

int tftb_tft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, int64_t* mults, int64_t* adds) {
    return host_tft_common(x, n, p, top, K, false, mults, adds);
}

int tftb_itft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, uint64_t inv2, int64_t* mults,
                  int64_t* adds) {
    if (inv2 != (p + 1) / 2) return fail("inv2 must be (p+1)/2");
    return host_tft_common(x, n, p, top, K, true, mults, adds);
}

int tftb_multiply_u64(const uint64_t* a, int64_t la, const uint64_t* b, int64_t lb, uint64_t* x, uint64_t p,
                      uint64_t top, int K, uint64_t inv2, int64_t* mults, int64_t* adds) {
    if (la <= 0 || lb <= 0) return fail("cannot multiply an empty polynomial");
    if (inv2 != (p + 1) / 2) return fail("inv2 must be (p+1)/2");
    const int64_t r = la + lb - 1;
    if (K < 62 && r > (1ll << K)) return fail("product length exceeds 2^K");
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    CtxLease lease;
    if (lease.acquire()) return -1;
    cudaStream_t st = lease.stream();
    const size_t wb = rh->wbytes;
    // device: a, b, x and the Y scratch as ring words, plus (u32 rings) a
    // bounded u64 staging for the conversions
    const size_t words = (size_t)(la + lb + 2 * r);
    const size_t wbytes = (words * wb + 255) & ~(size_t)255;
    const int64_t sw = wb == 4 ? std::min<int64_t>(std::max(la + lb, r), kStageWords) : 0;
    Scratch buf;
    if (buf.get(wbytes + (size_t)sw * 8, st)) return -1;
    uint64_t* stage = (uint64_t*)((char*)buf.p + wbytes);
    // pinned staging for pageable callers: [a | b | x]
    const size_t words64 = (size_t)(la + lb + r);
    const uint64_t* ha = a;
    const uint64_t* hb = b;
    uint64_t* hx = x;
    if (words64 * 8 <= kPinMax && !(host_pinned(a) && host_pinned(b) && host_pinned(x))) {
        if (lease.c->pin_reserve(words64 * 8)) return -1;
        uint64_t* hp = (uint64_t*)lease.c->pin;
        memcpy(hp, a, (size_t)la * 8);
        memcpy(hp + la, b, (size_t)lb * 8);
        ha = hp;
        hb = hp + la;
        hx = hp + la + lb;
    }
    int rc;
    if (wb == 4) {
        uint32_t* da = (uint32_t*)buf.p;
        uint32_t* db = da + la;
        uint32_t* dx = db + lb;
        uint32_t* dy = dx + r;
        if (upload_words(da, ha, la, stage, st) || upload_words(db, hb, lb, stage, st)) return -1;
        rc = rh->kind == 0 ? dispatch_mul<F30>(rh, da, la, la, db, lb, lb, dx, r, 1, dy, st)
                           : dispatch_mul<F32>(rh, da, la, la, db, lb, lb, dx, r, 1, dy, st);
        if (rc) return rc;
        if (download_words(hx, dx, r, stage, st)) return -1;
    } else {
        uint64_t* da = (uint64_t*)buf.p;
        uint64_t* db = da + la;
        uint64_t* dx = db + lb;
        uint64_t* dy = dx + r;
        if (upload_words(da, ha, la, stage, st) || upload_words(db, hb, lb, stage, st)) return -1;
        rc = dispatch_mul<F62>(rh, da, la, la, db, lb, lb, dx, r, 1, dy, st);
        if (rc) return rc;
        if (download_words(hx, dx, r, stage, st)) return -1;
    }
    CK(cudaStreamSynchronize(st));
    if (hx != x) memcpy(x, hx, (size_t)r * 8);
    tally_multiply(la, lb, p, K, mults, adds);
    return 0;
}

}  // extern "C"

namespace {

// Host-batch pipeline.  The vectors (sorted by offset, non-overlapping) are
// cut into sub-batches of consecutive vectors; sub-batch b runs on pipeline
// slot b mod 3, each slot a stream with its own device staging of one
// sub-batch: H2D of the sub-batch's vectors, packed back to back (one copy
// per run of touching vectors -- words between vectors are never read or
// written), u64 -> word conversion, the batch transform, conversion back,
// D2H of the same runs.  PCIe traffic in both directions overlaps the
// kernels of neighbouring sub-batches, and device memory is three
// sub-batches' staging whatever the batch size.
constexpr int kPipeStreams = 3;

cudaStream_t* pipe_streams() {
    static std::mutex mu;
    static std::map<int, std::vector<cudaStream_t>> per_dev;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto& v = per_dev[dev];
    if (v.empty()) {
        v.resize(kPipeStreams);
        for (auto& st : v) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    }
    return v.data();
}
std::mutex g_pipe_mu;  // one host-batch pipeline at a time per process (its streams are shared)

struct SubBatch {
    int64_t v0, v1;                                // [v0, v1) in sorted order
    int64_t words;                                 // packed words
    std::vector<std::pair<int64_t, int64_t>> runs;  // (host word offset, words), packed in order
};

template <class F>
int host_batch_pipeline(const RingHost* rh, uint64_t* x, const std::vector<int64_t>& ord, const int64_t* off,
                        const int64_t* len, int inverse) {
    using W = typename F::W;
    const bool narrow = sizeof(W) == 4;
    const int64_t count = (int64_t)ord.size();
    int64_t total = 0;
    for (int64_t i = 0; i < count; i++) total += len[ord[i]];
    // sub-batches of ~total/48 words (at least 2^22, at most 2^25 words
    // unless one vector is longer): short pipeline fill and drain
    // (measured: 12 -> 48 parts, +2% e2e)
    static const int parts = getenv("TFTB_PIPE_PARTS") ? atoi(getenv("TFTB_PIPE_PARTS")) : 48;      // A/B knobs
    static const int minlog = getenv("TFTB_PIPE_MINLOG") ? atoi(getenv("TFTB_PIPE_MINLOG")) : 22;
    const int64_t target = std::min<int64_t>(std::max<int64_t>(total / parts, 1ll << minlog), 1 << 25);
    std::vector<SubBatch> subs;
    int64_t maxw = 0;
    for (int64_t i0 = 0; i0 < count;) {
        SubBatch sb;
        sb.v0 = i0;
        sb.words = 0;
        int64_t i1 = i0;
        while (i1 < count && (sb.words < target || i1 == i0)) {
            const int64_t v = ord[i1];
            if (!sb.runs.empty() && sb.runs.back().first + sb.runs.back().second == off[v])
                sb.runs.back().second += len[v];
            else
                sb.runs.push_back({off[v], len[v]});
            sb.words += len[v];
            i1++;
        }
        sb.v1 = i1;
        maxw = std::max(maxw, sb.words);
        subs.push_back(std::move(sb));
        i0 = i1;
    }
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    cudaStream_t* ss = pipe_streams();
    // per-slot staging: u64 words (+ the word copy for u32 rings)
    const size_t slot_bytes = ((size_t)maxw * (narrow ? 12 : 8) + 255) & ~(size_t)255;
    Scratch buf;
    if (buf.get(slot_bytes * kPipeStreams, ss[0])) return -1;
    cudaEvent_t ready;
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, ss[0]));
    for (int i = 1; i < kPipeStreams; i++) CK(cudaStreamWaitEvent(ss[i], ready, 0));
    // Each sub-batch's plan is built as its turn comes, its arrays allocated
    // and uploaded stream-ordered on the slot's stream: the host runs ahead
    // of the copies instead of building all plans (an allocation and a
    // blocking upload each) before the first transfer starts.
    std::vector<std::unique_ptr<PlanImpl>> plans;
    std::vector<int64_t> poff, plen;
    auto make = [&](const SubBatch& sb, cudaStream_t st) -> int {
        poff.clear();
        plen.clear();
        int64_t acc = 0;
        for (int64_t i = sb.v0; i < sb.v1; i++) {
            poff.push_back(acc);
            plen.push_back(len[ord[i]]);
            acc += len[ord[i]];
        }
        plans.emplace_back(new PlanImpl());
        // (no forking: the pipeline's slots already overlap sub-batches, and
        // per-plan side streams would cost a stream creation per sub-batch)
        return plan_create<F>(rh, sb.v1 - sb.v0, 0, 0, poff.data(), plen.data(), plans.back().get(), st, true, false);
    };
    int rc = 0;
    for (size_t b = 0; b < subs.size() && !rc; b++) {
        const SubBatch& sb = subs[b];
        cudaStream_t st = ss[b % kPipeStreams];
        uint64_t* d64 = (uint64_t*)((char*)buf.p + slot_bytes * (b % kPipeStreams));
        W* dw = narrow ? (W*)(d64 + maxw) : (W*)d64;
        int64_t at = 0;
        for (auto& r : sb.runs) {
            if (cudaMemcpyAsync(d64 + at, x + r.first, (size_t)r.second * 8, cudaMemcpyHostToDevice, st)) rc = -1;
            at += r.second;
        }
        if (make(sb, st)) {
            rc = -1;
            break;
        }
        const int nb = (int)std::min<int64_t>((sb.words + 255) / 256, 148 * 8);
        if (narrow) {
            k_u64_to_w<W><<<nb, 256, 0, st>>>(d64, dw, sb.words);
            g_launches++;
        }
        if (!rc && plan_exec<F>(plans[b].get(), dw, inverse, nullptr, st)) rc = -1;
        if (narrow) {
            k_w_to_u64<W><<<nb, 256, 0, st>>>(dw, d64, sb.words);
            g_launches++;
        }
        at = 0;
        for (auto& r : sb.runs) {
            if (cudaMemcpyAsync(x + r.first, d64 + at, (size_t)r.second * 8, cudaMemcpyDeviceToHost, st)) rc = -1;
            at += r.second;
        }
        if (rc && g_err.empty()) fail(std::string("host batch copy: ") + cudaGetErrorString(cudaGetLastError()));
    }
    // the staging is released on slot 0 after every slot's work
    for (int i = 1; i < kPipeStreams; i++) {
        CK(cudaEventRecord(ready, ss[i]));
        CK(cudaStreamWaitEvent(ss[0], ready, 0));
    }
    for (int i = 0; i < kPipeStreams; i++) CK(cudaStreamSynchronize(ss[i]));
    cudaEventDestroy(ready);
    return rc;
}

}  // namespace

extern "C" {

int tftb_tft_batch_u64(uint64_t* x, const int64_t* off, const int64_t* len, int64_t count, uint64_t p,
                       uint64_t top, int K, int inverse) {
    if (count <= 0) return 0;
    if (!len || !x) return fail("x and len must not be NULL");
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    std::vector<int64_t> o(count);
    int64_t acc = 0;
    bool sorted = true;
    for (int64_t v = 0; v < count; v++) {
        if (len[v] <= 0 || (K < 62 && len[v] > (1ll << K))) return fail("vector length outside [1, 2^K]");
        o[v] = off ? off[v] : acc;
        if (o[v] < 0) return fail("negative vector offset");
        if (v && o[v] < o[v - 1]) sorted = false;
        acc += len[v];
    }
    std::vector<int64_t> ord(count);
    for (int64_t v = 0; v < count; v++) ord[v] = v;
    if (!sorted) std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return o[a] < o[b]; });
    for (int64_t i = 1; i < count; i++)
        if (o[ord[i]] < o[ord[i - 1]] + len[ord[i - 1]]) return fail("vectors overlap");
    switch (rh->kind) {
        case 0: return host_batch_pipeline<F30>(rh, x, ord, o.data(), len, inverse);
        case 1: return host_batch_pipeline<F32>(rh, x, ord, o.data(), len, inverse);
        default: return host_batch_pipeline<F62>(rh, x, ord, o.data(), len, inverse);
    }
}

struct tftb_ring {
    RingHost* h;
};

int tftb_ring_get(uint64_t p, uint64_t top, int K, tftb_ring** out) {
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    static std::mutex mu;
    static std::map<RingHost*, std::unique_ptr<tftb_ring>> handles;
    std::lock_guard<std::mutex> lk(mu);
    auto& h = handles[rh];
    if (!h) h.reset(new tftb_ring{rh});
    *out = h.get();
    return 0;
}

int tftb_ring_word_bytes(const tftb_ring* ring) { return ring ? ring->h->wbytes : -1; }

}  // extern "C"

namespace {
// Layout checks of the device batch entry points (tftbt200.h: vectors must
// not overlap): offsets >= 0, lengths in [1, 2^K], stride >= n.
int check_layout(const RingHost* rh, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                 const int64_t* h_len) {
    if (count < 0) return fail("negative vector count");
    const int64_t maxn = rh->K < 62 ? (1ll << rh->K) : INT64_MAX;
    if (!h_off && !h_len) {
        if (count > 0 && (n <= 0 || n > maxn)) return fail("vector length outside [1, 2^K]");
        if (count > 1 && stride < n) return fail("stride shorter than the vector length (vectors overlap)");
        return 0;
    }
    std::vector<std::pair<int64_t, int64_t>> iv(count);
    for (int64_t v = 0; v < count; v++) {
        const int64_t o = h_off ? h_off[v] : v * stride;
        const int64_t l = h_len ? h_len[v] : n;
        if (l <= 0 || l > maxn) return fail("vector length outside [1, 2^K]");
        if (o < 0) return fail("negative vector offset");
        iv[v] = {o, l};
    }
    std::sort(iv.begin(), iv.end());
    for (int64_t v = 1; v < count; v++)
        if (iv[v].first < iv[v - 1].first + iv[v - 1].second) return fail("vectors overlap");
    return 0;
}
}  // namespace

extern "C" {

int tftb_tft_dev(const tftb_ring* ring, void* data, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                 const int64_t* h_len, int inverse, void* stream) {
    if (!ring) return fail("null ring");
    const RingHost* rh = ring->h;
    if (check_layout(rh, count, n, stride, h_off, h_len)) return -1;
    if (count > 0 && !data) return fail("null data");
    cudaStream_t st = (cudaStream_t)stream;
    switch (rh->kind) {
        case 0: return dispatch_tft<F30>(rh, data, count, n, stride, h_off, h_len, inverse, st);
        case 1: return dispatch_tft<F32>(rh, data, count, n, stride, h_off, h_len, inverse, st);
        default: return dispatch_tft<F62>(rh, data, count, n, stride, h_off, h_len, inverse, st);
    }
}

struct tftb_plan {
    PlanImpl impl;
    int kind;
};

int tftb_plan_create(const tftb_ring* ring, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                     const int64_t* h_len, tftb_plan** out) {
    if (!ring || !out) return fail("null ring / out");
    if (count <= 0) return fail("plan needs at least one vector");
    const RingHost* rh = ring->h;
    if (check_layout(rh, count, n, stride, h_off, h_len)) return -1;
    std::unique_ptr<tftb_plan> pl(new tftb_plan());
    pl->kind = rh->kind;
    int rc = rh->kind == 0 ? plan_create<F30>(rh, count, n, stride, h_off, h_len, &pl->impl, nullptr, false)
             : rh->kind == 1 ? plan_create<F32>(rh, count, n, stride, h_off, h_len, &pl->impl, nullptr, false)
                             : plan_create<F62>(rh, count, n, stride, h_off, h_len, &pl->impl, nullptr, false);
    if (rc) return rc;
    *out = pl.release();
    return 0;
}

int tftb_plan_execute(const tftb_plan* plan, void* data, int inverse, void* stream) {
    if (!plan) return fail("null plan");
    cudaStream_t st = (cudaStream_t)stream;
    switch (plan->kind) {
        case 0: return plan_exec<F30>(&plan->impl, data, inverse, nullptr, st);
        case 1: return plan_exec<F32>(&plan->impl, data, inverse, nullptr, st);
        default: return plan_exec<F62>(&plan->impl, data, inverse, nullptr, st);
    }
}

int tftb_plan_destroy(tftb_plan* plan) {
    delete plan;
    return 0;
}

int tftb_multiply_dev(const tftb_ring* ring, const void* a, int64_t la, int64_t sa, const void* b, int64_t lb,
                      int64_t sb, void* x, int64_t sx, int64_t count, void* scratch, void* stream) {
    if (!ring) return fail("null ring");
    if (la <= 0 || lb <= 0) return fail("cannot multiply an empty polynomial");
    if (count < 0) return fail("negative pair count");
    if (count > 1 && (sa < la || sb < lb)) return fail("operand strides shorter than the operands");
    const RingHost* rh = ring->h;
    if (rh->K < 62 && la + lb - 1 > (1ll << rh->K)) return fail("product length exceeds 2^K");
    cudaStream_t st = (cudaStream_t)stream;
    switch (rh->kind) {
        case 0: return dispatch_mul<F30>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
        case 1: return dispatch_mul<F32>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
        default: return dispatch_mul<F62>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
    }
}

int tftb_words_from_u64(const tftb_ring* ring, const uint64_t* d_src, void* d_dst, int64_t n, void* stream) {
    if (!ring) return fail("null ring");
    cudaStream_t st = (cudaStream_t)stream;
    if (ring->h->wbytes == 8) {
        CK(cudaMemcpyAsync(d_dst, d_src, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (nb < 1) nb = 1;
    k_u64_to_w<uint32_t><<<nb, 256, 0, st>>>(d_src, (uint32_t*)d_dst, n);
    g_launches++;
    CK(cudaGetLastError());
    return 0;
}

int tftb_words_to_u64(const tftb_ring* ring, const void* d_src, uint64_t* d_dst, int64_t n, void* stream) {
    if (!ring) return fail("null ring");
    cudaStream_t st = (cudaStream_t)stream;
    if (ring->h->wbytes == 8) {
        CK(cudaMemcpyAsync(d_dst, d_src, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (nb < 1) nb = 1;
    k_w_to_u64<uint32_t><<<nb, 256, 0, st>>>((const uint32_t*)d_src, d_dst, n);
    g_launches++;
    CK(cudaGetLastError());
    return 0;
}

const char* tftb_last_error(void) { return g_err.c_str(); }
const char* tftb_version(void) { return "tftb200 0.1.0 (sm_100a)"; }
int64_t tftb_launch_count(int reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

int64_t tftb_stage_bytes(int reset) {
    const int64_t v = g_stage_peak;
    if (reset) g_stage_peak = g_stage_cur;
    return v;
}

int64_t tftb_aux_bytes(int reset) {
    const int64_t v = g_aux_peak;
    if (reset) g_aux_peak = g_aux_cur;
    return v;
}

int tftb_tally_transform(int64_t n, uint64_t p, int K, int inverse, int64_t* mults, int64_t* adds) {
    if (n <= 0) return fail("cannot tally an empty transform");
    tally_transform(n, p, K, inverse != 0, mults, adds);
    return 0;
}

int tftb_tally_multiply(int64_t la, int64_t lb, uint64_t p, int K, int64_t* mults, int64_t* adds) {
    if (la <= 0 || lb <= 0) return fail("cannot tally an empty product");
    tally_multiply(la, lb, p, K, mults, adds);
    return 0;
}

}  // extern "C"

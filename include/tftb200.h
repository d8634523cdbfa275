/*
 * tftb200 — B200-native in-place truncated Fourier transform (TFT), inverse
 * TFT and TFT-based polynomial product over Z/pZ (Harvey & Roche,
 * arXiv 1001.5272).  C ABI of libtftb200.so (sm_100a).
 *
 * Drop-in boundary.  The reference's native boundary is the Cython module
 * `tftmul._kernels`, selected by `tftmul.backend.kernels()`
 * (reference pkg/src/tftmul/backend.py:27-54) and called from
 * transforms.tft / itft / fft_pow2 (transforms.py:218-223, 232-236, 251-255)
 * and polymul.multiply (polymul.py:131-140).  The three host-pointer entry
 * points below replace its three functions one for one (same word type —
 * canonical uint64 residues —, same argument meaning, same in-place
 * contract, same (mults, adds) out-pair); they stage the words to the GPU,
 * run there, and copy back.  The kernels never raise in the reference
 * (`noexcept nogil`); here a negative status reports a CUDA or argument
 * failure and tftb_last_error() describes it.  There is no CPU fallback.
 *
 * Device-resident batched entry points (tftb_*_dev) take device buffers in
 * the ring's word type (uint32 when p < 2^32, uint64 otherwise) and a CUDA
 * stream; they are what the multi-GPU sharded benchmark and the torch-facing
 * Python API use.
 */
#ifndef TFTB200_H
#define TFTB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Replaces `_kernels.tft(u64[::1] x, long long off, long long n, u64 p, u64 top, int K)`
 * (reference _kernels.pyx:415-421): forward TFT of x[0:n) in place.
 * x: host pointer to n canonical residues (< p).  p odd prime < 2^62,
 * top = omegaK of exact order 2^K, n <= 2^K.  *mults/*adds (may be NULL)
 * receive the device algorithm's modular multiplication / addition counts. */
int tftb_tft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K,
                 int64_t* mults, int64_t* adds);

/* Replaces `_kernels.itft(x, off, n, p, top, K, inv2)` (_kernels.pyx:424-430):
 * inverse TFT of x[0:n) in place; inv2 must equal (p+1)/2. */
int tftb_itft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, uint64_t inv2,
                  int64_t* mults, int64_t* adds);

/* Replaces `_kernels.multiply(a, b, x, p, top, K, inv2)` (_kernels.pyx:433-480):
 * x[0:la+lb-1) = a * b mod p; a and b are read only; r = la+lb-1 <= 2^K. */
int tftb_multiply_u64(const uint64_t* a, int64_t la, const uint64_t* b, int64_t lb,
                      uint64_t* x, uint64_t p, uint64_t top, int K, uint64_t inv2,
                      int64_t* mults, int64_t* adds);

/* Batched host-buffer form of tftb_tft_u64 / tftb_itft_u64 (inverse != 0):
 * `count` vectors inside one host buffer x (uint64 words), vector v at
 * x + off[v] with length len[v] (host arrays; off == NULL -> back to back).
 * One H2D copy, one batched device transform, one D2H copy.  The reference
 * has no batch call — callers thread over buffers (nogil, _kernels.pyx:419);
 * this is that loop moved onto the device.  Pinned x gives full PCIe rate. */
int tftb_tft_batch_u64(uint64_t* x, const int64_t* off, const int64_t* len, int64_t count,
                       uint64_t p, uint64_t top, int K, int inverse);

/* Replaces `polymul.horner_eval(poly, point, cfg)` (reference polymul.py:39-52;
 * its compiled twin `horner_k`, _kernels.pyx:401-412): *out = sum_i poly[i]
 * point^i mod p over n >= 1 canonical host words, evaluated on the device
 * (segment Horner per thread, block reduction). */
int tftb_horner_u64(const uint64_t* poly, int64_t n, uint64_t point, uint64_t p, uint64_t* out);

/* Replaces `polymul.fold_twist(src, X, base, L, q, cfg)` (reference
 * polymul.py:55-88; `fold_twist_k`, _kernels.pyx:366-398): X[i mod L] +=
 * src[i] w^i for i < ls (X = the host block X + base, L words, w = omega(q);
 * w = 1 for q = 0), on the device. */
int tftb_fold_twist_u64(const uint64_t* src, int64_t ls, uint64_t* X, int64_t L, uint64_t w, uint64_t p);

/* ---------------------------------------------------------------- rings */
typedef struct tftb_ring tftb_ring;

/* Per-(p, omegaK, K) device twiddle tables (size independent of n; built
 * once, cached).  Same validity contract as RingConfig (modring.py:75-107);
 * the caller validates.  Returns 0 or a negative status. */
int tftb_ring_get(uint64_t p, uint64_t top, int K, tftb_ring** out);
/* bytes per device word for this ring: 4 (p < 2^32) or 8 */
int tftb_ring_word_bytes(const tftb_ring* ring);

/* ------------------------------------------------------ device batches */
/* In-place forward (inverse != 0: inverse) TFT of `count` vectors stored in
 * one device buffer `data` (ring word type).  Vector v starts at word
 * h_off[v] (or v*stride when h_off == NULL) and has length h_len[v] (or n
 * when h_len == NULL).  h_off/h_len are HOST arrays.  Vectors must not
 * overlap.  Words are canonical residues (< p), as everywhere in the
 * reference (modring.py:408-422); outputs are canonical.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Asynchronous w.r.t. the
 * host. */
int tftb_tft_dev(const tftb_ring* ring, void* data, int64_t count, int64_t n, int64_t stride,
                 const int64_t* h_off, const int64_t* h_len, int inverse, void* stream);

/* Reusable batch plan: the grouping of `count` vectors (same layout
 * arguments as tftb_tft_dev) by kernel plan, with its device-side offset /
 * length arrays and scratch allocated once.  Executing a plan issues only
 * kernel launches (no host synchronisation), so it can be captured in a
 * CUDA graph. */
typedef struct tftb_plan tftb_plan;
int tftb_plan_create(const tftb_ring* ring, int64_t count, int64_t n, int64_t stride,
                     const int64_t* h_off, const int64_t* h_len, tftb_plan** out);
int tftb_plan_execute(const tftb_plan* plan, void* data, int inverse, void* stream);
int tftb_plan_destroy(tftb_plan* plan);

/* Products of `count` pairs: x_v[0:la+lb-1) = a_v * b_v.  a_v = a + v*sa,
 * b_v = b + v*sb, x_v = x + v*sx (device words, ring word type).  `scratch`
 * is a device buffer of count*(la+lb-1) words (or NULL: allocated from the
 * stream-ordered pool).  a and b are never written. */
int tftb_multiply_dev(const tftb_ring* ring, const void* a, int64_t la, int64_t sa,
                      const void* b, int64_t lb, int64_t sb, void* x, int64_t sx,
                      int64_t count, void* scratch, void* stream);

/* Convert between host-API uint64 words and the ring's device word type on
 * the device (n words). */
int tftb_words_from_u64(const tftb_ring* ring, const uint64_t* d_src, void* d_dst, int64_t n,
                        void* stream);
int tftb_words_to_u64(const tftb_ring* ring, const void* d_src, uint64_t* d_dst, int64_t n,
                      void* stream);

/* ------------------------------------------------------------ misc */
const char* tftb_last_error(void);
const char* tftb_version(void);
/* Number of kernel launches issued by this thread since the last reset. */
int64_t tftb_launch_count(int reset);
/* Footprint audit (the device analogue of the reference's audited_call,
 * oracle.py:118-137): high-water mark of the device bytes this thread's
 * calls allocated beyond the transformed words themselves (two-pass stash,
 * p2r partial sums, the product's second operand) since the last reset.
 * Host-API staging of the caller's own words is not counted.  0 for every
 * transform with n <= 2^17 (u32 words): the tile and cluster plans run in
 * the n-word buffer alone. */
int64_t tftb_aux_bytes(int reset);

/* High-water mark of the device bytes this thread's host-pointer calls
 * (tftb_tft_u64 / tftb_itft_u64 / tftb_multiply_u64 / tftb_tft_batch_u64)
 * allocated for the caller's words since the last reset: the ring words
 * (4 B per word for p < 2^32) plus a bounded conversion staging (32 MB per
 * call, three sub-batches for the host batch), not 12 B per word. */
int64_t tftb_stage_bytes(int reset);

/* ------------------------------------------------------------ op tallies
 * (mults, adds) the reference walk reports for the same call: the second
 * tuple element of _kernels.tft / _kernels.itft (_kernels.pyx:415-430) and
 * of _kernels.multiply (_kernels.pyx:433-480).  Host-only (no GPU needed);
 * tftb_tft_u64 / tftb_itft_u64 / tftb_multiply_u64 return the same values. */
int tftb_tally_transform(int64_t n, uint64_t p, int K, int inverse, int64_t* mults, int64_t* adds);
int tftb_tally_multiply(int64_t la, int64_t lb, uint64_t p, int K, int64_t* mults, int64_t* adds);

#ifdef __cplusplus
}
#endif
#endif /* TFTB200_H */

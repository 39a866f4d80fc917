/*
 * raid6c.h -- C ABI of the B200-native Z_p-RAID library (libraid6c.so).
 *
 * Method: "An approach to RAID-6 based on cyclic groups" (arxiv cs/0611109).  A stripe is
 * N data strips d_0..d_{N-1} plus two parity strips P and Q.  Each strip is an LSB-first
 * bit stream of (p-1)-bit words, word w = stream bits [w(p-1), (w+1)(p-1)), bit j of a word
 * = coefficient of x^j of an element of R_p = F2[x]/(1 + x + ... + x^{p-1})
 * (Sec. 4.5; readings R1, R2).
 *
 *   P = d_0 + d_1 + ... + d_{N-1},   Q = d_0 + x d_1 + ... + x^{N-1} d_{N-1}
 *       (Eq. (znparity), Corollary 24.4; 0-based as Eq. (rsparity),
 *        PAPER.md:831-834; multiplication by x is the Sylvester matrix)
 *
 * and any two lost strips are rebuilt from the other N (Lemma 23.2, PAPER.md:370-406;
 * Sec. 4.3/4.6).
 *
 * Conventions for every call:
 *   - Strip indices: 0..N-1 data, N = P, N+1 = Q (R4).
 *   - Data strips are `bytes` long.  P and Q are raid6c_parity_bytes(p, bytes) long: the
 *     data are zero-extended to W = ceil(8*bytes/(p-1)) whole words and the parity holds all
 *     W*(p-1) bits; parity bits past W*(p-1) are written as zero (R5).
 *   - p is an odd prime, 3 <= p <= 257 (R7); 1 <= N <= 2p-1 data
 *     strips.  N <= p is the code of Eq. (znparity).  p < N <= 2p-1 is the extended code of
 *     Eq. (qext): data strip k >= p has Q-coefficient 1 + x^{k-p+1}; it is
 *     accepted only when p satisfies Theorem 25.3 (raid6c_ext_supported), else E_INVALID_N.
 *   - Pointers named "device" must be CUDA device memory of the plan's device; the caller
 *     owns all strip memory (the library never allocates or frees it).  A plan owns only
 *     small device/pinned work buffers, freed by raid6c_plan_destroy.
 *   - Lost strips are outputs: their input contents are never read.  All other strips are
 *     read-only inputs.  A recovered data strip is written for exactly `bytes` bytes.
 *   - Argument errors are returned synchronously, before any launch, with no side effect.
 *     Device-side failures are sticky and reported by raid6c_sync (and by the synchronous
 *     convenience calls).  There is no CPU fallback: every byte is computed by the
 *     library's sm_100a kernels.
 *   - Plan calls are stream-ordered on the plan's stream and return before completion.
 *     A plan is not thread-safe; distinct plans are independent.
 *   - Any alignment is accepted.  The TMA fast path needs every strip base and stride
 *     16-byte aligned; otherwise the (slower) direct-load path of the same kernel runs.
 */
#ifndef RAID6C_H
#define RAID6C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define RAID6C_MAX_P 257
#define RAID6C_MAX_STRIPS (2 * RAID6C_MAX_P + 1) /* 2p-1 data strips (extended code) + P + Q */

typedef enum {
    RAID6C_OK = 0,
    RAID6C_E_INVALID_P = 1,     /* p is not an odd prime in [3, 257] */
    RAID6C_E_INVALID_N = 2,     /* N < 1, N > 2p-1, or p < N with p failing Theorem 25.3 */
    RAID6C_E_INVALID_INDEX = 3, /* lost index outside [0, N+2) (lost_j: or RAID6C_NONE), or lost_i == lost_j */
    RAID6C_E_NULL = 4,          /* a required pointer is NULL */
    RAID6C_E_SIZE = 5,          /* bytes == 0, num_stripes < 0, or a stride smaller than its strip */
    RAID6C_E_CUDA = 6,          /* CUDA runtime / launch error (sticky; see raid6c_last_cuda_error) */
    RAID6C_E_NO_DEVICE = 7,     /* no CUDA device, or the device is not sm_100 */
    RAID6C_E_PLAN = 8           /* plan/call mismatch (p, N or bytes differ from the plan) */
} raid6c_status;

/* lost_j of a SINGLE erasure (the optional case of SPEC.md:441): only strip lost_i is lost.  The
 * library runs it as the pair (lost_i, Q) -- (P, Q) when lost_i is Q -- i.e. a lost data strip is
 * the XOR of the other data strips and P (Eq. (znparity), row 1), and the pair's parity strip is
 * regenerated from the data: the caller must let that INTACT parity strip be rewritten (with the
 * bytes it already holds when the stripe was consistent).  Accepted in the HOST arguments of
 * raid6c_recover, raid6c_recover_strided and raid6c_recover_host; every other call, and a DEVICE
 * array, must name two strips (RAID6C_E_INVALID_INDEX otherwise, where the library can see it). */
#define RAID6C_NONE (-1)

/* One erasure pair per stripe for batched recovery (either order; lost_j may be RAID6C_NONE in a
 * HOST array, never in a DEVICE array). */
typedef struct {
    int32_t lost_i;
    int32_t lost_j;
} raid6c_erasure;

typedef struct raid6c_plan_s *raid6c_plan;

/* ---------------------------------------------------------------- sizes (host only) */

/* W = ceil(8*bytes/(p-1)), the number of ring words per strip (R5).
 * Returns 0 for an invalid p. */
size_t raid6c_word_count(int p, size_t bytes);

/* Parity strip length ceil(W*(p-1)/8) bytes (R5).  0 for an invalid p. */
size_t raid6c_parity_bytes(int p, size_t bytes);

/* 1 if p is accepted (odd prime in [3,257]), else 0. */
int raid6c_valid_p(int p);

/* 1 if p runs the TMA fast-path kernel (the 28 primes whose period lcm(p-1, 32) fits 32 lanes),
   0 if it runs the generic kernel (the other 26 odd primes <= 257). */
int raid6c_has_fast_path(int p);

/* 1 if p satisfies Theorem 25.3: gcd(X^p + 1, X^m + X + 1) = 1 for all
 * 0 < m < p, so the extended code (up to 2p-1 data strips) recovers every pair.  Fails for the
 * Mersenne primes and 73 among p <= 257. */
int raid6c_ext_supported(int p);

/* Static description of the status code (never NULL). */
const char *raid6c_status_string(raid6c_status s);

/* Text of the last CUDA error seen by this thread (empty string if none). */
const char *raid6c_last_cuda_error(void);

/* Number of kernels this process has launched through the library (all plans). */
uint64_t raid6c_launch_count(void);

/* ---------------------------------------------------------------- plans */

/* Create a plan for (p, N, bytes) on CUDA device `device`, ordering work on `stream`
 * (a cudaStream_t; NULL = the legacy default stream).  The plan validates p and N once,
 * selects the kernel (fast or generic) and owns its small work buffers.  For the extended code
 * (N > p) it also builds, once, the solve multiplier of every erasure pair (C(N+2,2) entries of
 * 520 bytes on the device; host ring inversions -- about 0.6 s and 69 MB for p = 257, N = 513),
 * so recoveries never need a host round trip, even with device-resident erasure pairs. */
raid6c_status raid6c_plan_create(raid6c_plan *out, int p, int N, size_t bytes, int device, void *stream);
raid6c_status raid6c_plan_destroy(raid6c_plan plan);
raid6c_status raid6c_plan_set_stream(raid6c_plan plan, void *stream);

/* Wait for all work of the plan's stream; returns the first sticky error (and clears it). */
raid6c_status raid6c_sync(raid6c_plan plan);

/* ------------------------------------------- north-star single-stripe calls (synchronous) */

/* Encode one stripe on the current CUDA device (Eq. (znparity); Eq. (qext)
 * when N > p).
 * strips: HOST array of N DEVICE pointers (data strips, `bytes` each);  P, Q: DEVICE
 * pointers of raid6c_parity_bytes(p, bytes).  Synchronous: returns after the kernel has
 * completed, with its status. */
raid6c_status raid6c_encode(int p, int N, const uint8_t *const *strips, uint8_t *P, uint8_t *Q, size_t bytes);

/* Rebuild lost strips lost_i and lost_j (any order; lost_j = RAID6C_NONE: lost_i alone, see
 * RAID6C_NONE for the parity strip that is rewritten with it) of one stripe (Lemma 23.2,
 * PAPER.md:370-406; Sec. 4.6).  strips: HOST array of N+2 DEVICE
 * pointers, 0..N-1 data (`bytes`), N = P, N+1 = Q (parity_bytes).  The two lost strips are
 * written, the rest read.  Synchronous. */
raid6c_status raid6c_recover(int p, int N, int lost_i, int lost_j, uint8_t *const *strips, size_t bytes);

/* ------------------------------------------------ batched, stream-ordered device calls */

/* Encode num_stripes stripes.  Data strip k of stripe s is at
 *   data + s*stripe_stride + k*strip_stride            (DEVICE, `bytes` long)
 * and its parity at  P + s*parity_stride,  Q + s*parity_stride  (DEVICE, parity_bytes).
 * Requires strip_stride >= bytes, stripe_stride >= N*strip_stride (or num_stripes == 1),
 * parity_stride >= parity_bytes unless num_stripes == 1. */
raid6c_status raid6c_encode_strided(raid6c_plan plan, const uint8_t *data, size_t strip_stride,
                                    size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                    size_t parity_stride, int num_stripes);

/* Recover num_stripes stripes in place (same layout as raid6c_encode_strided): for stripe s
 * the strips named by erasures[s] (or erasures[0] for every stripe when num_erasures == 1)
 * are rebuilt from the other N strips of that stripe.  `erasures` is a HOST array when
 * erasures_on_device == 0, else a DEVICE array (already validated by the caller: each pair
 * distinct and in [0, N+2)).  Stripes may mix erasure classes (DD, DP, DQ, PQ).
 * Kernel choice (results are identical): a HOST list whose every pair is {P, Q} runs as an
 * encode (the PQ rebuild is Eq. (znparity) itself); a HOST list with no data-data pair runs
 * on the light recovery kernel (DP / DQ / PQ epilogues only; fast path, N <= p); anything
 * else, and every DEVICE list, on the full recovery kernel.  raid6c_recover chooses alike. */
raid6c_status raid6c_recover_strided(raid6c_plan plan, uint8_t *data, size_t strip_stride,
                                     size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                     size_t parity_stride, int num_stripes,
                                     const raid6c_erasure *erasures, int num_erasures,
                                     int erasures_on_device);

/* ------------------------------------------------ around the path */

/* Scrub: check both parity equations of Eq. (znparity) on every word of
 * num_stripes stripes (same layout as raid6c_encode_strided; all strips are read, none
 * written).  bad_words: DEVICE array of num_stripes uint32; entry s is overwritten with the
 * number of words w of stripe s for which P_w != sum_i d_{i,w} or Q_w != sum_i x^i d_{i,w}.
 * Stream-ordered. */
raid6c_status raid6c_scrub_strided(raid6c_plan plan, const uint8_t *data, size_t strip_stride,
                                   size_t stripe_stride, const uint8_t *P, const uint8_t *Q,
                                   size_t parity_stride, int num_stripes, uint32_t *bad_words);

/* Small write: in stripe s, data strip k_s (disks[s], or disks[0] for every stripe when
 * num_disks == 1; 0 <= k_s < N) is replaced by the `bytes` at new_data + s*new_stride
 * (DEVICE), and P, Q are updated in the same pass by linearity of Eq. (znparity):
 *   P' = P + (d_k + d_k'),   Q' = Q + x^k (d_k + d_k').
 * Reads old d_k, new d_k, P, Q; writes d_k, P, Q.  `disks` is HOST memory unless
 * disks_on_device != 0 (then a DEVICE int32 array, already validated).  Stream-ordered.
 * new_data must not overlap the stripe. */
raid6c_status raid6c_update_strided(raid6c_plan plan, uint8_t *data, size_t strip_stride,
                                    size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                    size_t parity_stride, int num_stripes, const uint8_t *new_data,
                                    size_t new_stride, const int32_t *disks, int num_disks,
                                    int disks_on_device);

/* ------------------------------------------------ comparison system */

/* The paper's comparison system, Reed-Solomon RAID-6 over GF(2^8) (Sec. 4.1-4.4,
 * PAPER.md:818-1039): P = sum D_i, Q = sum g^i D_i with g = {02} and reduction polynomial
 * x^8+x^4+x^3+x^2+1 (Eq. (rsparity)); recovery per Sec. 4.3.  1 <= N <= 255 data strips; every
 * strip (data, P, Q) is `bytes` long.  Same layout, pointer and error conventions as the
 * strided Z_p calls; stream-ordered on `stream` (a cudaStream_t, NULL = legacy default). */
raid6c_status raid6c_rs_encode_strided(int N, size_t bytes, const uint8_t *data, size_t strip_stride,
                                       size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                       size_t parity_stride, int num_stripes, void *stream);
raid6c_status raid6c_rs_recover_strided(int N, size_t bytes, uint8_t *data, size_t strip_stride,
                                        size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                        size_t parity_stride, int num_stripes,
                                        const raid6c_erasure *erasures, int num_erasures,
                                        int erasures_on_device, void *stream);

/* ------------------------------------ cross-GPU stripe layout */

/* The strips of one stripe may live on different GPUs ("ranks"): rank r holds the strips
 * with global index in a contiguous range [k_lo, k_hi) of 0..N+1.  Both parity equations of
 * Eq. (znparity) are sums over disks, and the reduction pi of
 * R' = F2[x]/(x^p+1) -> R_p is a ring homomorphism (Eq. (powers)), so the
 * syndromes split into per-rank partial sums of already-reduced words, and the recovery
 * syndromes of Eq. (PQxy) likewise:
 *
 *   dP = sum_r dP_r,   dQ = sum_r dQ_r,   dP_r, dQ_r = the surviving strips of rank r only.
 *
 * A step is two launches per rank with a cross-rank barrier between them:
 *   1. raid6c_partial_strided: rank r folds its local surviving strips into (dP_r, dQ_r)
 *      (HBM-bound, the same TMA pipeline as encode) and stores word range g of the result
 *      into part_p[g] / part_q[g] -- a slot owned by rank g, local or a peer pointer
 *      (NVLink stores, overlapped with the fold tile by tile).
 *   2. raid6c_combine_strided: rank g XORs the num_sources partial slots of its word range
 *      (in the owner's memory; peer pointers are accepted too) and applies the class solve of
 *      Lemma 23.2 / Sec. 4.6 in the same kernel, writing the
 *      rebuilt strips (or P and Q for an encode) straight to their owners (peer pointers).
 *
 * Encode is the PQ case: pass erasures == NULL.  Word ranges: the parity-format strip
 * (parity_bytes) is cut into ranges of raid6c_xgpu_range_bytes(p, bytes, G) bytes, range g =
 * [g*range_bytes, min((g+1)*range_bytes, parity_bytes)); a range is a whole number of kernel
 * tiles, so no tile straddles two owners.  Every pointer below is a DEVICE address valid on
 * the plan's device (its own memory, or peer memory mapped with raid6c_ipc_open / peer
 * access).  The two launches never wait on each other inside a kernel: ordering across
 * ranks is the caller's barrier (stream-ordered collective or host barrier). */

#define RAID6C_MAX_RANKS 64

/* Word-range size for num_ranks owners of (p, bytes) stripes: a multiple of p's kernel tile
 * (fast path) or byte group (generic path) such that num_ranks ranges cover parity_bytes.
 * Host only.  0 on bad input. */
size_t raid6c_xgpu_range_bytes(int p, size_t bytes, int num_ranks);

/* Partial syndromes of the local strips.  strips: HOST array of N+2 DEVICE pointers indexed
 * by global strip index; only [k_lo, k_hi) are read (others may be NULL).  Strip k of stripe
 * s is at strips[k] + s*(k < N ? data_stride : parity_stride).  erasures: as in
 * raid6c_recover_strided (host or device array of 1 or num_stripes pairs), or NULL for an
 * encode.  Lost strips are not read.  Output for stripe s, word range g (bytes
 * [g*range_bytes, ...) of the parity-format strip):
 *   part_p[g] + s*part_stride + (off - g*range_bytes) <- dP_r bytes at offset off
 *   part_q[g] + ...                                     <- dQ_r (reduced, rotation origin at
 *                                                          the lost strip for DP/DD)
 * part_p / part_q: HOST arrays of num_ranges DEVICE pointers; range_bytes from
 * raid6c_xgpu_range_bytes(p, bytes, num_ranges); part_stride >= range_bytes when num_stripes > 1.
 * Stream-ordered on the plan's stream. */
raid6c_status raid6c_partial_strided(raid6c_plan plan, const uint8_t *const *strips, size_t data_stride,
                                     size_t parity_stride, int num_stripes, const raid6c_erasure *erasures,
                                     int num_erasures, int erasures_on_device, int k_lo, int k_hi,
                                     int num_ranges, uint8_t *const *part_p, uint8_t *const *part_q,
                                     size_t part_stride, size_t range_bytes);

/* Combine + solve for bytes [range_lo, range_hi) of every stripe (range_lo a multiple of the
 * range granule; range_hi a multiple of it too, or equal to parity_bytes -- anything else is
 * RAID6C_E_SIZE, since the kernels work in whole granules).  src_p / src_q: HOST arrays of num_sources DEVICE
 * pointers; source r holds stripe s's partial of this range at src_p[r] + s*part_stride.
 * strips: HOST array of N+2 DEVICE pointers (global index, strides as in the partial call);
 * only the two output strips of each stripe are written (lost strips; P and Q for an
 * encode), clipped to their length (`bytes` for data, parity_bytes for P/Q).  erasures must
 * equal the partial call's.  Stream-ordered on the plan's stream. */
raid6c_status raid6c_combine_strided(raid6c_plan plan, uint8_t *const *strips, size_t data_stride,
                                     size_t parity_stride, int num_stripes, const raid6c_erasure *erasures,
                                     int num_erasures, int erasures_on_device, int num_sources,
                                     const uint8_t *const *src_p, const uint8_t *const *src_q,
                                     size_t part_stride, size_t range_lo, size_t range_hi);

/* Inter-process device memory for the cross-GPU layout (one process per GPU).
 * raid6c_dev_alloc: cudaMalloc'd buffer on `device` (exportable; freed by raid6c_dev_free).
 * raid6c_ipc_export: 64-byte CUDA IPC handle of a buffer from raid6c_dev_alloc.
 * raid6c_ipc_open: map a peer's handle into this process on `device` (enables peer access
 * to the owning device when it differs); close with raid6c_ipc_close. */
raid6c_status raid6c_dev_alloc(size_t bytes, int device, void **dev_ptr);
raid6c_status raid6c_dev_free(void *dev_ptr);
raid6c_status raid6c_ipc_export(const void *dev_ptr, uint8_t handle[64]);
raid6c_status raid6c_ipc_open(const uint8_t handle[64], int device, void **dev_ptr);
raid6c_status raid6c_ipc_close(void *dev_ptr);

/* ------------------------------------------------ host-buffer calls (end-to-end path) */

/* Same as the strided calls, but every pointer is HOST memory (pinned memory gives
 * full-duplex PCIe overlap; pageable memory works but is slower).  The plan streams the
 * stripes through its own device staging ring: H2D copy, kernel and D2H copy of
 * successive chunks overlap on separate streams.  Synchronous: returns when the results
 * are in host memory.  For recovery only the surviving strips are copied in and only
 * the two rebuilt strips of each stripe are copied out. */
raid6c_status raid6c_encode_host(raid6c_plan plan, const uint8_t *data, size_t strip_stride,
                                 size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                 size_t parity_stride, int num_stripes);
raid6c_status raid6c_recover_host(raid6c_plan plan, uint8_t *data, size_t strip_stride,
                                  size_t stripe_stride, uint8_t *P, uint8_t *Q,
                                  size_t parity_stride, int num_stripes,
                                  const raid6c_erasure *erasures, int num_erasures);

/* Bytes moved host->device and device->host by the last *_host call on this plan. */
raid6c_status raid6c_host_traffic(raid6c_plan plan, uint64_t *h2d_bytes, uint64_t *d2h_bytes);

/* ------------------------------------------------ harness kernels (not the method) */

/* Fill DEVICE strips with the synthetic generator of synthetic/gen.py (DESIGN.md "input
 * recipe"): for s in [0, nstripes), t in [0, nstrips) the `len` bytes at
 * dst + s*stripe_stride + t*strip_stride get strip (strip0 + t) of stripe (stripe0 + s) of
 * config `cfg`.  sparse_mode: 0 uniform, 1 sparse (each byte 0 with probability 0.9),
 * 2 sparse for odd global stripe indices only (config 4).  Stream-ordered on `stream`. */
raid6c_status raid6c_fill(uint8_t *dst, size_t strip_stride, size_t stripe_stride, size_t len, int nstrips,
                          int nstripes, uint64_t seed, int cfg, int stripe0, int strip0, int sparse_mode,
                          void *stream);

/* Count mismatching bytes between two DEVICE buffers; the count is added to *count_dev
 * (a DEVICE uint64).  Stream-ordered. */
raid6c_status raid6c_count_mismatch(const uint8_t *a, const uint8_t *b, size_t len,
                                    uint64_t *count_dev, void *stream);

/* Per-strip 64-bit digests of DEVICE strips (test / bench harness, not the method; host
 * version: synthetic/digest.py).  For s in [0, nstripes), t in [0, nstrips), the `len` bytes at
 * src + s*stripe_stride + t*strip_stride get
 *   digests_dev[s*nstrips + t] = mix64(len ^ 0xBB67AE8584CAA73B)
 *                                + sum_k mix64(w_k + k*0x9E3779B97F4A7C15 + 0x6A09E667F3BCC909)  (mod 2^64),
 * w_k the little-endian u64 of bytes [8k, 8k+8) (zero past len), mix64 = SplitMix64's finalizer.
 * A changed word always changes the digest (mix64 is a bijection), so equal digests of a GPU
 * strip and an oracle strip computed elsewhere stand for equal bytes (up to 2^-64 per pair).
 * digests_dev is a DEVICE array of nstrips*nstripes uint64, overwritten.  Stream-ordered. */
raid6c_status raid6c_digest(const uint8_t *src, size_t strip_stride, size_t stripe_stride, size_t len,
                            int nstrips, int nstripes, uint64_t *digests_dev, void *stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RAID6C_H */

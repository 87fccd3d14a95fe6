/*
 * smgpu.h -- C ABI of the B200-native exact string-matching hot path of
 *   Tarhio, Holub, Giaquinta, "Technology Beats Algorithms (in Exact String
 *   Matching)", arXiv:1612.01506.
 *
 * The problem (Sec. 1): "counting or reporting all the locations
 * of given pattern p of length m=|p| in given text t of length n=|t|", p and t
 * strings over a finite alphabet.  Here the alphabet is all 256 byte values;
 * NUL is an ordinary symbol (reading R15).  The argument order (p, m, t, n)
 * follows Naive-search(p, m, t, n), PAPER.md:41 (Alg. 1).
 *
 * Result definition (Alg. 1; every alignment is visited, so
 * occurrences overlap, reading R3):
 *      count = #{ i in [0, n-m] : t[i..i+m) == p }           (0 if n < m)
 * Positions are 0-based byte offsets (paper position - 1, reading R1),
 * reported strictly ascending = Alg. 1's loop order.
 *
 * Method (Algs. 3-4): pattern positions are compared in
 * the order pi of increasing frequency of their symbol in the text
 * (PAPER.md:16,113,138), the first r comparisons unconditionally ("loop
 * peeling"), blocks of alignments dropped as soon as no
 * alignment in them survives.  Order, peeling factor and
 * strategy change the work done, never the result.
 *
 * Placement and ownership
 *   - t, d_hist, d_count, pos: DEVICE memory of the current CUDA device.
 *     t is checked with cudaPointerGetAttributes; host memory is rejected
 *     with SM_EINVAL (there is no CPU fallback).
 *   - p, order, hist: HOST memory, read during the call only (the pattern
 *     and its order are packed into kernel parameters at launch).
 *   - The caller owns every buffer; the library keeps no pointer after the
 *     call returns (async calls: after the enqueued work completes).
 *   - Scratch comes from the library's own stream-ordered memory pool per
 *     device (cudaMemPoolCreate; freed blocks stay cached, up to
 *     SMGPU_POOL_KEEP_BYTES if set, until sm_trim_scratch); the device's
 *     default pool is not touched.
 *   - stream: a cudaStream_t passed as void*; NULL means cudaStreamPerThread.
 *
 * Errors: every call except sm_count returns sm_status and records it (with a
 * message) in thread-local state readable by sm_last_error()/
 * sm_last_error_message().  sm_count returns SM_COUNT_ERROR on failure.
 *   SM_EINVAL  m == 0, m > SM_MAX_PATTERN, NULL p with m > 0, NULL t with n > 0,
 *              t not device memory, bad strategy/order.
 *   n < m (including n == 0) is NOT an error: count 0 (reading R2).
 *   SM_ETRUNC  sm_report found more than cap occurrences (first cap written).
 *   SM_ECUDA   a CUDA runtime error (message has the CUDA error string).
 *
 * Re-entrancy: no global mutable state besides the thread-local error; calls
 * on different streams may overlap.
 */
#ifndef SMGPU_H
#define SMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sm_status {
  SM_OK = 0,
  SM_EINVAL = 1,
  SM_ETRUNC = 2,
  SM_ENOMEM = 3,
  SM_ECUDA = 4
} sm_status;

/* Which device strategy evaluates the remaining comparisons (both exact):
 *  SM_STRATEGY_FILTER: the first comparison (pi(1), the rarest symbol) is done
 *     for 16 alignments per lane with packed-byte compares; each surviving
 *     alignment then runs pi(2..m) with early exit (alpha drops to 1 after
 *     the peeled block compare).  Best when the rarest symbol is rare.
 *  SM_STRATEGY_BLOCK: Alg. 4 as written: r peeled packed-byte compares over
 *     16 alignments per lane, then the pi-ordered loop over the warp's 512
 *     alignments with a warp-uniform exit test.  Best for
 *     small alphabets / periodic text.
 *  SM_STRATEGY_PACKED: BLOCK on b-bit codes (b = 1 or 2) of the text bytes,
 *     code(x) = (x >> s) & (2^b - 1) with s chosen so that the code is injective
 *     on the symbols present in t according to hist; needs <= 4 symbols in hist
 *     and every pattern symbol present in hist, else SM_EINVAL.
 *     For DNA / binary text (compare-bound regime).
 *     A caller histogram is ADVISORY (frequencies "computed in
 *     advance from some relevant corpus"): it steers order and strategy, never
 *     the result.  When a caller hist would select PACKED, counting packs the
 *     text once on the device and checks there that every byte of t is one of
 *     hist's symbols; if one is not, the PACKED launches yield on the device to
 *     byte-compare launches of the same patterns (BLOCK / PAIR / FILTER), with
 *     no host synchronisation.  Reporting instead takes order and strategy from
 *     t's own device histogram whenever a caller hist would allow PACKED.
 *  SM_STRATEGY_PAIR: FILTER with the rarest-two-symbol chunk test: a 16-byte
 *     chunk is queued only if one of its alignments matches pi(1) AND pi(2)
 *     (m >= 2; m = 1 runs FILTER).  Best when pi(1) is too frequent for
 *     FILTER's single-symbol chunk test to skip much.
 *  SM_STRATEGY_AUTO: chosen on the host from the text histogram. */
typedef enum sm_strategy {
  SM_STRATEGY_AUTO = 0,
  SM_STRATEGY_FILTER = 1,
  SM_STRATEGY_BLOCK = 2,
  SM_STRATEGY_PACKED = 3,
  SM_STRATEGY_PAIR = 4
} sm_strategy;

#define SM_COUNT_ERROR UINT64_MAX
#define SM_MAX_PATTERN 4096u

/* ------------------------------------------------------------------------ */
/* North-star calls (synchronous; run on cudaStreamPerThread)               */
/* ------------------------------------------------------------------------ */

/* Number of (overlapping) occurrences of p[0..m) in device text t[0..n).
 * Computes the text histogram and rarest-first order internally.
 * Returns SM_COUNT_ERROR (and sets sm_last_error) on failure. */
uint64_t sm_count(const uint8_t* p, size_t m, const uint8_t* t, size_t n);

/* Reporting version ("printing position i"): writes the first
 * min(count, cap) ascending 0-based positions to DEVICE array pos[0..cap) and
 * the total count to *count_out (host).  count > cap -> SM_ETRUNC (positions
 * beyond cap are dropped; *count_out is the total).  Two-call idiom: cap=0. */
sm_status sm_report(const uint8_t* p, size_t m, const uint8_t* t, size_t n,
                    uint64_t* pos, size_t cap, uint64_t* count_out);

/* Comparison order pi: order[k] (host, m entries) = 0-based
 * pattern position compared k-th; positions sorted by ascending count of
 * their symbol in t (device histogram), ties by ascending position (R11). */
sm_status sm_symbol_order(const uint8_t* t, size_t n, const uint8_t* p, size_t m,
                          uint32_t* order);

/* ------------------------------------------------------------------------ */
/* Building blocks (asynchronous unless stated)                              */
/* ------------------------------------------------------------------------ */

/* d_hist[c] = #{x in [0,n) : t[x] = c}, c = 0..255 (DEVICE u64[256],
 * overwritten).  Async on `stream`.  PAPER.md:16,113 (frequencies in the text). */
sm_status sm_histogram(const uint8_t* t, size_t n, uint64_t* d_hist, void* stream);

/* Host-only: stable rarest-first order from a host histogram. */
sm_status sm_order_from_histogram(const uint64_t* hist, const uint8_t* p, size_t m,
                                  uint32_t* order);

/* Enqueue the count of p in t on `stream`; the result lands in *d_count
 * (DEVICE u64, overwritten).
 *   hist     host u64[256] symbol frequencies for order and strategy (t's
 *            histogram, or another corpus's: advisory, see SM_STRATEGY_PACKED);
 *            NULL -> t's histogram computed on the device (synchronises `stream`).
 *   order    host u32[m] comparison order (any permutation of 0..m-1);
 *            NULL -> rarest-first from hist.
 *   peel     peeling factor r >= 1 (clamped to m, reading R9); 0 -> auto.
 *   strategy sm_strategy. */
sm_status sm_count_async(const uint8_t* p, size_t m, const uint8_t* t, size_t n,
                         const uint64_t* hist, const uint32_t* order, uint32_t peel,
                         int strategy, uint64_t* d_count, void* stream);

/* Enqueue the counts of P patterns p[i] (host, lengths m[i]) in one device text:
 * d_counts[i] (DEVICE u64[P], overwritten) = number of occurrences of p[i] starting
 * at alignments i < min(n - m[i] + 1, max_alignments) -- pass SIZE_MAX to count
 * all of them; a smaller value counts exactly the alignments a text shard owns
 * (the bytes past them are its halo).  Each pattern is still a
 * full pass over the text (no sharing of reads between patterns); batching only
 * lets the persistent kernel flow from one pattern's last tiles into the next
 * pattern's first tiles and amortises launch overhead.  hist: as in
 * sm_count_async; order and peeling factor are chosen per pattern (AUTO).
 * Scratch: for P >= 2 over a text with <= 4 distinct symbols the call packs the
 * text once into a temporary b-bit code array (b = 1 or 2; ~n b / 8 bytes from the
 * stream-ordered pool, freed on the stream) that the PACKED passes read instead of
 * the bytes (SMGPU_PREPACK=0 disables). */
sm_status sm_count_batch(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                         size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* d_counts,
                         void* stream);

/* sm_count_batch with the caller's comparison order and peeling factor per pattern
 * (NEXT-2's fixed orders, and r sweeps, on the
 * batched path): orders = host u32, the P orders concatenated (m[i] entries each, a
 * permutation of 0..m[i]-1; NULL -> rarest-first from hist), peels = host u32[P]
 * (0 or NULL -> auto).  Orders and r never change a count. */
sm_status sm_count_batch_ordered(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                                 size_t max_alignments, const uint64_t* hist, const uint32_t* orders,
                                 const uint32_t* peels, int strategy, uint64_t* d_counts, void* stream);

/* Multi-GPU counting without a collective call (NEXT-4, the counting
 * version, summed over ranks): as sm_count_batch, but mc_counts (u64[P]) is the NVLink
 * MULTICAST address of a buffer bound on every rank of the group (e.g. torch symmetric
 * memory's multicast_ptr, or cuMulticastCreate + cuMulticastBindMem).  The rank's
 * counts go to library scratch, and the last CTA to finish each search launch adds
 * its patterns' counts to mc_counts with one multimem.red each (NVLS: the switch
 * applies the add to every rank's bound copy) -- no extra kernel, no NCCL call.  When
 * all ranks' work has completed, every rank's own copy holds the sums over all ranks.
 * The call does NOT zero the counts: every rank zeroes its copy and the group
 * synchronises before any rank launches, and synchronises again (after its stream)
 * before reading.  Same p, m, max_alignments (each rank passes its shard's owned
 * alignments), hist and strategy as sm_count_batch.  SM_EINVAL for a misaligned
 * mc_counts.  SMGPU_NVLS_EMULATE=1 replaces multimem.red by a plain atomic add (a
 * unicast mc_counts: tests of the protocol on a box without multicast). */
sm_status sm_count_batch_multicast(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                                   size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* mc_counts,
                                   void* stream);

/* Enqueue the reporting version: the first min(count, cap) ascending
 * positions go to DEVICE pos[0..cap), the total count to DEVICE *d_count.
 * Truncation is detected by the caller (*d_count > cap) after the stream
 * synchronises.  Same hist/order/peel/strategy meaning as sm_count_async. */
sm_status sm_report_async(const uint8_t* p, size_t m, const uint8_t* t, size_t n,
                          const uint64_t* hist, const uint32_t* order, uint32_t peel,
                          int strategy, uint64_t* pos, size_t cap, uint64_t* d_count,
                          void* stream);

/* Enqueue the reporting version for P patterns (see sm_count_batch for p, m,
 * max_alignments, hist, strategy, and the code-array scratch).  One read of the text
 * per pattern: matches are staged compactly (scratch from the stream-ordered pool:
 * ~24 B per (pattern, 32 KiB tile) plus a staging pool of min(4 GiB, 64 MiB +
 * min(16 cap, 4.2 KiB per (pattern, tile)) + 38 KiB per SM per launch) bytes, mostly
 * untouched; SMGPU_STAGE_BYTES overrides), then expanded; tiles that do not fit the pool
 * are recomputed from the text -- never a different result.  d_counts[i] (DEVICE u64[P]) = count of p[i];
 * positions of all patterns are written CONCATENATED in pattern order into DEVICE
 * pos[0..cap): pattern i's ascending positions start at sum_{j<i} d_counts[j].
 * Positions past cap are dropped (the caller detects truncation from d_counts).
 * position_offset is added to every written position (0 for a whole text; a text
 * shard passes the global position of its first byte, so its positions are global). */
sm_status sm_report_batch(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                          size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* pos, size_t cap,
                          uint64_t* d_counts, uint64_t position_offset, void* stream);

/* Fixed comparison orders of PAPER.md:184-186 (Sec. 2.4), for the order ablation
 * (the paper's N / N-freq / N-fixed columns).  Host-only; order[m] out (0-based).
 *   SM_ORDER_IDENTITY: 0, 1, ..., m-1 (Algs. 1-2).
 *   SM_ORDER_PI_H:     p[1], p[m], p[4], p[7], ..., p[3], p[6], ..., p[2], p[5], ...
 *                      (1-based; stride-3 chains from 4, 3, 2, taken positions skipped).
 *   SM_ORDER_PI_HS:    pi_h over the non-`space` positions, then the `space` positions
 *                      ascending ("moving first all the spaces to the end").
 * The result is a permutation usable as `order` in sm_count_async / sm_report_async. */
typedef enum sm_order_kind { SM_ORDER_IDENTITY = 0, SM_ORDER_PI_H = 1, SM_ORDER_PI_HS = 2 } sm_order_kind;
sm_status sm_heuristic_order(const uint8_t* p, size_t m, int kind, uint8_t space, uint32_t* order);

/* Plan introspection (host-only, no GPU work): the strategy and peeling
 * factor sm_count_async would pick for (p, hist, order).  Used by tests and
 * the benchmark to label measurements. */
sm_status sm_plan(const uint8_t* p, size_t m, const uint64_t* hist, const uint32_t* order,
                  uint32_t peel, int strategy, int* strategy_out, uint32_t* peel_out);

/* Compare-step counters (NEXT-2 instrumentation; PAPER.md:34,176-178 discuss how many
 * comparisons the method executes).  Only the instrumented build libsmgpu_counters.so
 * (compiled with -DSMGPU_COUNTERS) counts; the release library returns SM_EINVAL.
 * Synchronises the device, copies the device-wide totals since the last reset into
 * out[0..8) (host) and, if reset != 0, zeroes them:
 *   out[0] (warp, work item) pairs processed
 *   out[1] BLOCK/PACKED warp-blocks (512 x CPL consecutive alignments) holding >= 1
 *          valid alignment -- Alg. 4's blocks at alpha = out[7]
 *   out[2] BLOCK/PACKED SIMDcompare steps executed in those blocks (peeled + loop)
 *   out[3] FILTER 16-alignment chunks whose pi(1)-bytes were tested
 *   out[4] FILTER chunks holding p[pi(1)]
 *   out[5] FILTER valid alignments matching pi(1) and pi(2)
 *   out[6] FILTER pattern positions compared while verifying those
 *   out[7] BLOCK/PACKED alignments per warp-block (max over launches)
 * (out: host u64[8]) */
sm_status sm_counters(uint64_t* out, int reset);

/* Thread-local status of the last failing call on this thread (SM_OK if none
 * since sm_clear_error), its message, and a static name for a status. */
sm_status sm_last_error(void);
const char* sm_last_error_message(void);
void sm_clear_error(void);
const char* sm_status_string(sm_status s);

/* Return the library's cached scratch memory on the current device to the driver,
 * keeping at most keep_bytes (0: all of it).  The pool caches freed per-call scratch
 * (reporting staging up to 4 GiB, code arrays) so repeated calls cost no remapping;
 * call this when that memory is needed elsewhere.  Synchronises the device. */
sm_status sm_trim_scratch(size_t keep_bytes);

/* Library version string and the number of kernels the library has launched
 * on this thread (for the benchmark's gpu_launches claim). */
const char* sm_version(void);
uint64_t sm_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SMGPU_H */

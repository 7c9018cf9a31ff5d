/*
 * pmh.h -- C ABI of the B200-native ProbMinHash signature engine (libpmh.so).
 *
 * Drop-in boundary for the reference's kernel layer
 *   /root/reference/pkg/src/probminhash/_kernels.py   (K)
 * which the reference's public API (sketch.py:121-213, estimate.py:91-123)
 * calls one set at a time as
 *   K._k_<algo>(ids: uint64[n], weights: float64[n], m) -> (uint64[m], int64[3])
 * and K._k_sketch_dispatch(algo_id, ids, weights, m) (K:884-917).
 * Here a call covers a whole CSR batch of sets; a single set is a batch of 1.
 *
 * Conventions: plain pointers and sizes only.  Functions named *_host take
 * host pointers and perform the host<->device copies themselves; all others
 * take DEVICE pointers, are stream-ordered on `stream` (a cudaStream_t, NULL =
 * legacy default stream) and synchronise that stream only to report errors.
 * Algorithm ids are the reference's ALG_* constants (K:866-881).
 * Return value: PMH_OK or a negative PMH_ERR_* code; *err_set (if non-NULL)
 * receives the index of the first offending set for EMPTY / RANDOMNESS.
 * Workspaces are stream-ordered allocations from the device's DEFAULT memory
 * pool; the first allocating call sets that pool's release threshold to
 * UINT64_MAX, so freed workspaces stay mapped for the next call instead of
 * being unmapped at every synchronisation (a caller sharing the default pool
 * keeps its freed memory cached too; cudaMemPoolTrimTo releases it).
 */
#ifndef PMH_H_
#define PMH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (errors.py:4-17) */
#define PMH_OK 0
#define PMH_ERR_EMPTY (-1)      /* EmptyInputError: a set has no elements   */
#define PMH_ERR_INVALID (-2)    /* InvalidParamsError: m / algo / b domain  */
#define PMH_ERR_RANDOMNESS (-3) /* RandomnessFailureError: loop cap hit      */
#define PMH_ERR_CUDA (-4)       /* CUDA runtime failure (see last_error)    */
#define PMH_ERR_NOMEM (-5)

/* algorithm ids, K:866-881 */
#define PMH_ALG_PMINHASH 0
#define PMH_ALG_PMH1 1
#define PMH_ALG_PMH1A 2
#define PMH_ALG_PMH2 3
#define PMH_ALG_PMH3 4
#define PMH_ALG_PMH3A 5
#define PMH_ALG_PMH4 6
#define PMH_ALG_MINHASH 10
#define PMH_ALG_SUPERMINHASH 11
#define PMH_ALG_OPH 12
#define PMH_ALG_UW1 13
#define PMH_ALG_UW1A 14
#define PMH_ALG_UW2 15
#define PMH_ALG_UW3 16
#define PMH_ALG_UW3A 17
#define PMH_ALG_UW4 18

/* library version (major*10000 + minor*100 + patch) */
int pmh_version(void);

/* human-readable description of the last error on this thread */
const char* pmh_last_error(void);

/*
 * Sketch a CSR batch of sets.
 * Replaces K._k_pminhash (K:284), _k_probminhash1/1a/2/3/3a/4 (K:303-614),
 * _k_uw_probminhash3/3a/4 (K:619-763) and the unit-weight calls of
 * sketch_unweighted (sketch.py:188-213), i.e. K._k_sketch_dispatch (K:884).
 *   ids       uint64[nelems]      element ids, set s = [offsets[s], offsets[s+1])
 *   weights   float64[nelems]     positive finite weights; ignored (may be NULL)
 *                                  for the unweighted algorithms (ids 13..18)
 *   offsets   int64[nsets+1]
 *   sig_out   uint64[nsets*m]     row-major signatures (element ids)
 *   stats_out int64[nsets*3] or NULL: [points generated, elements needing more
 *             than one point (interleaved variants 1a/3a only, else 0),
 *             successful slot updates] -- GPU-schedule statistics, see DESIGN.md
 * m >= 1 (m >= 2 for PMH3/3a/4 and UW3/3a/4, sketch.py:148-166,198).
 */
int pmh_sketch_csr(int algo, int64_t m, const uint64_t* ids,
                   const double* weights, const int64_t* offsets,
                   int64_t nsets, uint64_t* sig_out, int64_t* stats_out,
                   int64_t* err_set, void* stream);

/*
 * Asynchronous form: enqueue on `stream` without synchronising.  d_status is a
 * caller-owned DEVICE int64[2] initialised with pmh_status_reset(); device-side
 * failures (EMPTY / RANDOMNESS) accumulate there and are reported by
 * pmh_status_check(), which synchronises the stream.  Host-side argument
 * errors are returned immediately.  pmh_sketch_csr == reset + async + check.
 */
int pmh_sketch_csr_async(int algo, int64_t m, const uint64_t* ids,
                         const double* weights, const int64_t* offsets,
                         int64_t nsets, uint64_t* sig_out, int64_t* stats_out,
                         int64_t* d_status, void* stream);

/*
 * The same batch sketched by nalgos algorithms (sig_outs[k] / stats_outs[k]
 * for algos[k], device buffers; stats_outs or its entries may be NULL):
 * the variants run CONCURRENTLY on internal streams forked from and joined
 * back into `stream` (no host sync), so one kernel's tail overlaps the next
 * one's work.  Each signature equals the single-algorithm call's.  The
 * reference has no multi-algorithm call; this is the batched form of N calls
 * of K._k_sketch_dispatch (K:884-917) over the same input.
 */
int pmh_sketch_csr_multi_async(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                               const double* weights, const int64_t* offsets, int64_t nsets,
                               uint64_t* const* sig_outs, int64_t* const* stats_outs,
                               int64_t* d_status, void* stream);
/*
 * The asynchronous sketch with the sets' total weights KNOWN IN ADVANCE:
 * set_weights is a DEVICE float64[nsets] (W_s = sum of set s's weights), or
 * NULL to compute them.  This is the non-streaming form of ProbMinHash2/4
 * (BASELINE configs[3]; the reference has no non-streaming code): the kernels
 * skip their weight pre-pass and size the threshold guess from W_s.  Any
 * positive W_s gives the SAME signature (the final verification max_k h_k <=
 * guess makes every guess exact-safe; a wrong W_s only costs time).  Accepted
 * for every weighted algorithm; ignored by the unweighted ones.
 */
int pmh_sketch_csr_w_async(int algo, int64_t m, const uint64_t* ids, const double* weights,
                           const int64_t* offsets, int64_t nsets, const double* set_weights,
                           uint64_t* sig_out, int64_t* stats_out, int64_t* d_status,
                           void* stream);

/* Per-set total weights of a CSR batch (DEVICE buffers, stream-ordered):
 * out[s] = sum of weights[offsets[s] .. offsets[s+1]). */
int pmh_set_weights(const double* weights, const int64_t* offsets, int64_t nsets, double* out,
                    void* stream);

int pmh_status_reset(int64_t* d_status, void* stream);
int pmh_status_check(const int64_t* d_status, int64_t* err_set, void* stream);

/* Same with HOST buffers (pageable or pinned); nelems = offsets[nsets]. */
/*
 * Several algorithms over one host batch: the inputs cross PCIe once, in
 * set-chunks that the first algorithm consumes as they land; each algorithm's
 * signatures (sig_outs[k], host uint64[nsets*m]) and optional stats
 * (stats_outs[k] or NULL) are copied back while the next one computes.
 * Host-side empties are reported before any copy (EmptyInputError, *err_set).
 */
int pmh_sketch_csr_host_multi(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                              const double* weights, const int64_t* offsets, int64_t nsets,
                              int64_t nelems, uint64_t* const* sig_outs,
                              int64_t* const* stats_outs, int64_t* err_set);

/*
 * Enqueue-only form of pmh_sketch_csr_host_multi: returns once the work is
 * queued on internal streams, WITHOUT waiting for prior work on `stream`
 * (the inputs are host buffers); `stream` is made to wait for its completion
 * (copies back to the host buffers included).  Errors found while running
 * land in d_status, which must be reset and settled before the first call
 * (pmh_status_reset + a stream sync) and checked after the last.
 * Host buffers must stay valid and unmodified until `stream` has passed this
 * work, and should be pinned for the copies to overlap.  Consecutive calls
 * use different internal streams, so one batch's H2D overlaps the previous
 * batch's kernels (pipelined batches).
 */
int pmh_sketch_csr_host_multi_async(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                                    const double* weights, const int64_t* offsets, int64_t nsets,
                                    int64_t nelems, uint64_t* const* sig_outs,
                                    int64_t* const* stats_outs, int64_t* d_status, void* stream);
int pmh_sketch_csr_host(int algo, int64_t m, const uint64_t* ids,
                        const double* weights, const int64_t* offsets,
                        int64_t nsets, int64_t nelems, uint64_t* sig_out,
                        int64_t* stats_out, int64_t* err_set);

/*
 * Equal-component counts of npairs signature pairs (rows of A and B):
 * counts[p] = #{k : A[p,k] == B[p,k]}.  estimate_similarity (estimate.py:91-95)
 * is counts[p] / m.
 */
int pmh_count_equal(const uint64_t* a, const uint64_t* b, int64_t npairs,
                    int64_t m, int32_t* counts, void* stream);

/*
 * All-pairs tile over n signatures (row-major [n, m]): for rows i in [r0,r1)
 * and columns j in [c0,c1) with j > i, out[(i-r0)*ld + (j-c0)] = count(i,j).
 * Entries with j <= i are left untouched.
 */
int pmh_allpairs_tile(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0,
                      int64_t r1, int64_t c0, int64_t c1, uint16_t* out,
                      int64_t ld, void* stream);

/*
 * All-pairs reduction over rows [r0,r1) x cols [c0,c1) (pairs j > i): adds to
 * hist[c] (uint64[m+1], caller-zeroed) the number of pairs with c equal
 * components, and appends every pair with count >= thr to pairs as
 * {(i << 32) | j, count} (uint64[2*cap]); *cursor (caller-zeroed uint64)
 * ends at the number of such pairs (entries beyond cap are dropped; the
 * order of the list is unspecified).  thr >= 1 runs two exact stages (low-
 * word compares over every pair, 64-bit recount of the pairs with a low-word
 * match; a stream-ordered temporary of up to 32 MB from the device pool);
 * thr <= 0 lists every pair in one stage.
 */
int pmh_allpairs_hist(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0, int64_t r1,
                      int64_t c0, int64_t c1, int32_t thr, uint64_t* hist, uint64_t* pairs,
                      int64_t cap, uint64_t* cursor, void* stream);

/*
 * The same reduction by an exact hash join on (component, value)
 * (csrc/pmh_join.cuh): only the pairs sharing a component are ever visited,
 * so a batch whose sets rarely share components (configs[4]) costs O(n m)
 * instead of O(n^2 m).  Same histogram and pair set as pmh_allpairs_hist
 * (thr >= 1).  Synchronises the stream once (the work check).  Returns 1 --
 * nothing written -- when the pairs sharing a key exceed max_visits (<= 0:
 * 2^26; e.g. many duplicate sets) or thr <= 0; the caller then runs
 * pmh_allpairs_hist.  Stream-ordered temporaries from the device pool (up to
 * ~1.5 GB of tables plus the pair map).
 */
int pmh_allpairs_join_hist(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0, int64_t r1,
                           int64_t c0, int64_t c1, int32_t thr, uint64_t* hist, uint64_t* pairs,
                           int64_t cap, uint64_t* cursor, int64_t max_visits, void* stream);

/* b-bit reduction of nsets*m components (estimate.py:105-114, K:851-861). */
int pmh_bbit(const uint64_t* sig, int64_t nsets, int64_t m, int b,
             int64_t* out, void* stream);

/*
 * Packed b-bit signatures (the "popc-style" estimator of SURVEY §8f-1):
 * pmh_bbit_pack fuses the b-bit reduction (estimate.py:105-114, K:851-861)
 * with packing -- row s, word w holds components k = w*F + f (F = floor(64/b),
 * f < F) at bits [f*b, f*b + b), unused fields 0; pmh_bbit_words(m, b) =
 * ceil(m / F) words per row (-1 on bad arguments).
 * pmh_allpairs_bbit_hist is pmh_allpairs_hist over packed rows: hist[C] counts
 * the pairs (j > i) with C equal b-bit components; pairs with C >= thr are
 * appended.  The estimate of a pair is clamp((C/m - 2^-b)/(1 - 2^-b), 0, 1)
 * (estimate_similarity_bbit, estimate.py:117-123).
 */
int64_t pmh_bbit_words(int64_t m, int b);
int pmh_bbit_pack(const uint64_t* sig, int64_t nsets, int64_t m, int b, uint64_t* packed,
                  void* stream);
int pmh_allpairs_bbit_hist(const uint64_t* packed, int64_t n, int64_t m, int b, int64_t r0,
                           int64_t r1, int64_t c0, int64_t c1, int32_t thr, uint64_t* hist,
                           uint64_t* pairs, int64_t cap, uint64_t* cursor, void* stream);

/*
 * Fused MSE cell: replaces K._k_mse_cell(algo, m, wa, wb, seed, s) (K:920-963,
 * called by harness.run_mse_cell harness.py:266-280).  For each of s pairs
 * the ids come from ONE splitmix64 stream seeded with `seed` (pair t, weight
 * pair q -> word t*npairs + q), side A holds the q with wa[q] > 0, side B the
 * q with wb[q] > 0; both are sketched with `algo` at m and their equal
 * components counted into matches[t] (HOST int64[s]).  wa/wb are HOST
 * arrays.  Generation, sketching and counting run on the device in chunks;
 * synchronous on `stream`.  Errors as pmh_sketch_csr (an all-zero side ->
 * PMH_ERR_EMPTY).
 */
int pmh_mse_cell(int algo, int64_t m, const double* wa, const double* wb, int64_t npairs,
                 uint64_t seed, int64_t s, int64_t* matches, void* stream);

/*
 * Host ingestion of the reference CLI's "id weight" lines
 * (cli._read_weighted_lines, cli.py:60-70) into CSR arrays, no device work:
 * blank and '#' lines skipped, id = Python int(tok, 0) (non-negative, < 2^64),
 * weight = Python float(tok) or 1.0 when absent.  Returns the number of
 * entries, -(line number) of the first line outside that grammar (the caller
 * then falls back to the exact restatement for the reference's error),
 * -(2^62) if more than cap entries, -(2^61) on bad arguments.
 */
int64_t pmh_parse_weighted_text(const char* buf, int64_t len, uint64_t* ids, double* weights,
                                int64_t cap);

/*
 * Diagnostic: measured 32-bit ALU-pipe peak of the current device in Gop/s
 * (8 independent LOP3 chains per thread, full occupancy) -- the roofline
 * denominator for the integer-bound signature kernels.  Synchronous.
 */
int pmh_probe_alu_peak(double* gops_out, double* ms_out);

/* Pipe-peak microbenchmark of one instruction kind (0 = LOP3 / 32-bit ALU
 * pipe, 1 = IMAD / integer multiply-add, 2 = DFMA / FP64 pipe, 3 = FFMA / the
 * issue-slot ceiling): 8 independent chains per thread at full occupancy,
 * best of 5 launches on the legacy stream.  Thread-level ops per second in
 * *gops_out (10^9), the launch time in *ms_out.  Synchronous. */
int pmh_probe_pipe_peak(int kind, double* gops_out, double* ms_out);

/* Per-point work probe (csrc/pmh_probe.cuh): points/s (10^9) of a tight
 * loop generating ProbMinHash points with one splitmix64 word, the value
 * (kind 0: log1p, the ProbMinHash1/2 point; kind 1: TruncExp fast path, the
 * ProbMinHash3/4 point) and a 128-bit CAS offer into a shared 1024-slot
 * table, at full occupancy.  The practical point-rate ceiling that bench.py's
 * per-variant roofline divides by.  Synchronous. */
int pmh_probe_point_rate(int kind, double* gpts_out, double* ms_out);

/* The device build of the glibc log1p (fn 0) / expm1 (fn 1) restatements
 * (csrc/pmh_math.cuh; reference K:120-122, K:146), and (fn 2) the log1p
 * specialised to the sampled domain x = -U that the kernels call, evaluated on
 * n DEVICE doubles x into out (expm1: NaN where it reports no result).
 * Stream-ordered.  For parity tests of the transcendental itself. */
int pmh_math_eval(int fn, const double* x, int64_t n, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PMH_H_ */

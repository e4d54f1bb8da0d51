/*
 * aliasfft_b200.h — C ABI of the B200-native aliasing-filter sparse-FFT hot path.
 *
 * The reference (`aliasfft` 0.1.0, pure Python on numpy) has no FFI: its operator
 * API is the Python function surface re-exported by
 * /root/reference/pkg/src/aliasfft/__init__.py:9-79.  Each entry point below is the
 * device-side body of one of those functions (cited per function), with plain
 * pointers and sizes so any host language can bind it (see INTEGRATION.md for the
 * ctypes binding the Python mirror uses).
 *
 * Conventions
 *  - Every pointer named x/out/nodes/... is DEVICE memory unless marked (host).
 *    Small plan arrays (factors, shifts) are HOST arrays copied into kernel
 *    parameters; the library never reads device memory on the host.
 *  - Complex values are interleaved (re, im).  Signals may be complex64
 *    (AFFT_C64, float2) or complex128 (AFFT_C128, double2); all arithmetic after
 *    the gather is IEEE float64 with no FMA contraction, as numpy computes.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls only enqueue work, except those documented as synchronising.
 *  - Return codes: 0 OK, <0 error (AFFT_E*); afft_last_error() gives the
 *    thread-local message.  No exception crosses the ABI.
 *  - Batched layout: `batch` signals, signal s starting at x + s*ld elements.
 *  - Node layout (peeling graph, /root/reference/pkg/src/aliasfft/peeling.py:169-178):
 *    node g = (sum of factors before cycle c) + bucket index i, measurements
 *    contiguous per node: nodes[s][g][r], r over the shift list.
 */
#ifndef ALIASFFT_B200_H
#define ALIASFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum afft_dtype { AFFT_C64 = 0, AFFT_C128 = 1 };

enum afft_status {
  AFFT_OK = 0,
  AFFT_EINVAL = -1,       /* maps to ValueError */
  AFFT_EUNSUPPORTED = -2, /* maps to UnsupportedSizeError / ValueError */
  AFFT_ECUDA = -3,        /* CUDA launch/runtime failure */
  AFFT_ENOMEM = -4        /* workspace too small */
};

/* NodeState (peeling.py:29-34) as stored in the int8 state arrays. */
enum afft_node_state {
  AFFT_UNKNOWN = 0,
  AFFT_ZERO_TON = 1,
  AFFT_SINGLE_TON = 2,
  AFFT_MULTI_TON = 3,
  AFFT_RESOLVED = 4
};

#define AFFT_MAX_CYCLES 16
#define AFFT_MAX_SHIFTS 512
#define AFFT_MAX_SMEM_DFT 4096 /* largest bucket count handled by the one-CTA DFT */

const char* afft_last_error(void);
int afft_version(void);

/*
 * bucketize / bucketize_set (bucketize.py:83-106):
 *   out[s][t][i] = (1/b) * sum_j x_s[(j*(n/b) - shifts[t]) mod n] * exp(-2*pi*i*j*i/b)
 * Output strides (in complex elements) let one call write either the
 * FilteredSpectrum layout [s][t][i] or the node layout [s][i][t].
 */
int afft_bucketize(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                   int64_t b, const int64_t* shifts /* host */, int32_t nshift,
                   double* out, int64_t out_signal_stride, int64_t out_shift_stride,
                   int64_t out_bin_stride, void* stream);

/*
 * build_graph (peeling.py:169-178): all cycles and shifts in one launch, node layout
 * nodes[s][g][r] with g = cycle offset + bucket, r over shifts (stride nshift).
 */
int afft_build_graph(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                     const int64_t* factors /* host */, int32_t ncycles,
                     const int64_t* shifts /* host */, int32_t nshift, double* nodes,
                     void* stream);

/*
 * Per-signal sum of |x|^2 in float64, written as fixed-order partials
 * partials[s][p], p < afft_sumsq_parts(n, dtype).  The 2-norm used by
 * exact_thresholds (peeling.py:316-318) is sqrt(sum_p partials[s][p]).
 */
int32_t afft_sumsq_parts(int64_t n, int dtype);
int afft_sumsq(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
               double* partials, void* stream);

/* exact_thresholds (peeling.py:316-318) from the partials: eps[s] = 1e-6*||x_s||/sqrt(n). */
int afft_exact_thresholds(const double* partials, int32_t nparts, int64_t n, int64_t batch,
                          double* eps, void* stream);

/*
 * peel_decode, exact mode (peeling.py:270-313 with classify_exact 193-215 and
 * subtract 181-190).  One CTA per signal; synchronous rounds with first-found
 * dedupe in (cycle, bucket) order, subtraction in found order, ZERO_TON frozen.
 *   residual  [batch][nodes][3]  in/out (complex128)
 *   state     [batch][nodes]     in/out (afft_node_state)
 *   node_f0   [batch][nodes]     out (last decoded position, -1 if none)
 *   node_val  [batch][nodes]     out (complex128, last decoded value)
 *   eps_zero / eps_ratio [batch] per-signal thresholds
 *   rec_pos/rec_val [batch][rec_cap] in/out: recovered spectrum in insertion
 *     order; rec_count[s] on entry is the number already recovered.
 *   rounds/unresolved [batch] out.
 * node_f0/node_val may be NULL.
 */
int afft_peel_exact(int64_t n, int64_t batch, const int64_t* factors /* host */,
                    int32_t ncycles, double* residual, int8_t* state, int64_t* node_f0,
                    double* node_val, const double* eps_zero, const double* eps_ratio,
                    int32_t max_rounds, int64_t* rec_pos, double* rec_val, int32_t rec_cap,
                    int32_t* rec_count, int32_t* rounds, int32_t* unresolved, void* stream);

/*
 * The paper's Fig. 5 tree-walk ("sparse-graph decoder by packet erasure channel
 * method"; a non-goal of the reference) for exact mode:
 * every live node identified once, then paths extended from single-ton nodes through a
 * FIFO queue — each decoded tone is subtracted from its d check nodes and only those
 * are re-identified.  Same arguments and outputs as afft_peel_exact (recovered set equal
 * to the round decoder's; order the walk's); rounds[s] = the walk's generations,
 * identifications[s] (may be NULL) = check-node identifications performed.
 */
int afft_peel_tree_exact(int64_t n, int64_t batch, const int64_t* factors /* host */,
                         int32_t ncycles, double* residual, int8_t* state, int64_t* node_f0,
                         double* node_val, const double* eps_zero, const double* eps_ratio,
                         int64_t* rec_pos, double* rec_val, int32_t rec_cap,
                         int32_t* rec_count, int32_t* rounds, int32_t* unresolved,
                         int32_t* identifications, void* stream);

/*
 * classify_exact (peeling.py:193-215) for `count` independent nodes of one cycle
 * size b: residual [count][3] complex128, index [count] bucket indices.  Writes
 * state, and f0/val where the node is a SINGLE_TON (f0/val are in/out so a
 * node's last decode survives, like BucketNode.f0/.value).
 */
int afft_classify_exact(const double* residual, const int64_t* index, int64_t count, int64_t b,
                        int64_t n, double eps_zero, double eps_ratio, int8_t* state,
                        int64_t* f0, double* val, void* stream);

/*
 * subtract (peeling.py:186-190): residual[i][r] -= value[i] * exp(-2j*pi*((shifts[r]*f[i]) mod n)/n)
 * for `count` nodes with `nshift` measurements each (residue check is the caller's).
 */
int afft_subtract(double* residual, const int64_t* shifts /* host */, int32_t nshift,
                  const int64_t* f, const double* value, int64_t count, int64_t n,
                  void* stream);

/*
 * truncate_spectrum (oneshot.py:260-263): keep the k largest |v|, ties to the
 * smaller position; output sorted by that key.  out_count[s] = min(k, count[s]).
 */
int afft_truncate(const int64_t* pos, const double* val, const int32_t* count, int32_t cap,
                  int64_t batch, int32_t k, int64_t* out_pos, double* out_val,
                  int32_t* out_count, void* stream);

/*
 * truncate_spectrum (oneshot.py:260-263) of one HOST entry list (the native DSFFT loop's
 * output): the min(k, count) largest |v| (hypot, as numpy's abs), ties to the smaller
 * position, written in that order to out_pos/out_val (host).  Runs on the calling
 * thread without touching the device (the Python drop-in calls it per signal with the
 * GIL released, instead of a numpy lexsort under the GIL).
 */
int afft_truncate_host(const int64_t* pos, const double* val, int64_t count, int32_t k,
                       int64_t* out_pos, double* out_val, int64_t* out_count);

/* Resident ffast_fused_kernel CTAs per SM and its dynamic shared memory for a plan. */
int afft_ffast_occupancy(int64_t n, const int64_t* factors /* host */, int32_t ncycles,
                         int32_t* blocks_per_sm /* host */, int32_t* smem_bytes /* host */);

/*
 * ffast (peeling.py:321-332) over a batch with an explicit cycle plan and the
 * exact shift set (0,1,2): fused norm → thresholds → build_graph → peel → truncate.
 * Workspace: afft_ffast_workspace_size bytes of device memory.
 *   out_pos/out_val [batch][k] (truncated, sorted by (-|v|, f)), out_count [batch]
 *   all_pos/all_val [batch][sum factors] pre-truncation spectrum (may be NULL)
 *   all_count, rounds, unresolved [batch] (may be NULL)
 * max_rounds <= 0 means k + 4 (peeling.py:330).
 */
size_t afft_ffast_workspace_size(int64_t n, int dtype, int64_t batch,
                                 const int64_t* factors /* host */, int32_t ncycles);
int afft_ffast(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
               const int64_t* factors /* host */, int32_t ncycles, int32_t k,
               int32_t max_rounds, int64_t* out_pos, double* out_val, int32_t* out_count,
               int64_t* all_pos, double* all_val, int32_t* all_count, int32_t* rounds,
               int32_t* unresolved, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ R-FFAST (noisy) */

/* Node energies ||vec_e||^2 over `nshift` measurements each (peeling.py:354-357). */
int afft_node_energies(const double* vec, int32_t nshift, int64_t count, double* energy,
                       void* stream);

/*
 * robust_thresholds (peeling.py:335-351) per signal over `count` energies:
 * sigma = sqrt(median(E[mask]) / r), floor = 1e-8 * sqrt(max E),
 * t0 = max(1.5 sigma sqrt(r), floor), t1 = max(2.5 sigma sqrt(r), floor).
 * mask [batch][count] selects the median's reference set (NULL = all; an empty
 * set falls back to all, dsfft.py:164-166).
 */
int afft_robust_thresholds(const double* energy, const uint8_t* mask, int64_t count,
                           int64_t batch, int32_t r, double* t0, double* t1, void* stream);

/*
 * One huge R-FFAST decode across ranks (SURVEY §8(e) stretch row): every rank holds the
 * whole graph and the same state; the singleton search's candidate chunks are split
 * round-robin over the ranks, and once per round `exchange` must replace each of the
 * `count` partial slots (score double, candidate int32, on the device, stream-ordered on
 * `stream`) by its minimum over all ranks — e.g. two NCCL all-reduces with op MIN.
 * Slots a rank did not scan hold (+inf, INT32_MAX).  Returns 0 on success.  Results are
 * identical to the single-rank decode.
 */
typedef int (*afft_exchange_fn)(void* ctx, double* part_score, int32_t* part_t, int64_t count,
                                void* stream);
typedef struct {
  int32_t rank, world;
  afft_exchange_fn exchange;
  void* ctx;
} AfftSearchShard;

int afft_peel_noisy_sharded(int64_t n, int64_t batch, const int64_t* factors /* host */,
                            int32_t ncycles, const int64_t* shifts /* host */, int32_t nshift,
                            int32_t c, int32_t m, const double* weights /* host */,
                            double* residual, int8_t* state, int64_t* node_f0, double* node_val,
                            const double* t0, const double* t1, int32_t max_rounds,
                            int64_t* rec_pos, double* rec_val, int32_t rec_cap,
                            int32_t* rec_count, int32_t* rounds, int32_t* unresolved,
                            void* workspace, size_t workspace_bytes, void* stream,
                            const AfftSearchShard* shard);

/* Workspace bytes for afft_peel_noisy / (with batch = node count) the per-node search. */
size_t afft_noisy_workspace_size(int64_t n, int64_t batch, const int64_t* factors /* host */,
                                 int32_t ncycles, int32_t c, int32_t m);

/* Workspace bytes for afft_singleton_search_noisy / afft_classify_noisy over `count` nodes. */
size_t afft_singleton_workspace_size(int64_t n, int64_t count, int64_t b, int32_t c, int32_t m);

/*
 * singleton_search_noisy (peeling.py:222-250) for `count` nodes of one cycle size b:
 * residual [count][c*m], index [count]; shifts (host) = SearchPlan.shifts, weights
 * (host) = kay_weights(m).  Outputs f0, val (complex128), resnorm per node.
 * Workspace: afft_singleton_workspace_size(n, count, b, c, m).  Stream-ordered.
 */
int afft_singleton_search_noisy(const double* residual, const int64_t* index, int64_t count,
                                int64_t b, int64_t n, const int64_t* shifts, int32_t nshift,
                                int32_t c, int32_t m, const double* weights, int64_t* f0,
                                double* val, double* resnorm, void* workspace,
                                size_t workspace_bytes, void* stream);

/* classify_noisy (peeling.py:253-267) for `count` nodes: search + the t0/t1 gates. */
int afft_classify_noisy(const double* residual, const int64_t* index, int64_t count, int64_t b,
                        int64_t n, const int64_t* shifts, int32_t nshift, int32_t c, int32_t m,
                        const double* weights, double t0, double t1, int8_t* state,
                        int64_t* f0, double* val, double* resnorm, void* workspace,
                        size_t workspace_bytes, void* stream);

/*
 * peel_decode, noisy mode (peeling.py:270-313 with classify_noisy 253-267) over a
 * batch of graphs in node layout residual[s][g][c*m]: rounds of
 * prep -> exhaustive search -> fit -> harvest/subtract on the device, the round loop
 * itself a CUDA-graph WHILE node whose condition the last kernel of each round sets
 * (no host round-trip; stream-ordered).  t0/t1 [batch] per-signal gates.
 * State/f0/val/rec_* as in afft_peel_exact.  The sharded variant (one signal's search
 * split over ranks) exchanges partials through the host callback once per round and
 * synchronises.
 */
int afft_peel_noisy(int64_t n, int64_t batch, const int64_t* factors /* host */, int32_t ncycles,
                    const int64_t* shifts /* host */, int32_t nshift, int32_t c, int32_t m,
                    const double* weights /* host */, double* residual, int8_t* state,
                    int64_t* node_f0, double* node_val, const double* t0, const double* t1,
                    int32_t max_rounds, int64_t* rec_pos, double* rec_val, int32_t rec_cap,
                    int32_t* rec_count, int32_t* rounds, int32_t* unresolved, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * r_ffast (peeling.py:361-386) over a batch, one stream-ordered enqueue: build_graph
 * at each signal's own search shifts (SearchPlan.shifts = anchors[j] + 2^j t,
 * peeling.py:60-62; anchors [batch][c] host, row stride anchor_stride, 0 = one set for
 * every signal) -> node energies -> robust_thresholds (peeling.py:335-358) -> noisy
 * peel_decode with max_rounds (0: k + 4, peeling.py:384) -> truncate_spectrum.
 * weights (host, m - 1) = kay_weights(m).  Outputs (device): out_* [batch][k]
 * truncated, all_* [batch][sum factors] the pre-truncation spectrum in insertion
 * order, rounds / unresolved / t0 / t1 [batch].  Workspace: afft_rffast_workspace_size.
 * Replaces the reference's per-signal r_ffast call (peeling.py:361) and its
 * build_graph / noisy_thresholds / peel_decode sequence.
 */
size_t afft_rffast_workspace_size(int64_t n, int64_t batch, const int64_t* factors /* host */,
                                  int32_t ncycles, int32_t c, int32_t m);
int afft_rffast(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                const int64_t* factors /* host */, int32_t ncycles,
                const int64_t* anchors /* host */, int64_t anchor_stride, int32_t c, int32_t m,
                const double* weights /* host */, int32_t k, int32_t max_rounds, int64_t* out_pos,
                double* out_val, int32_t* out_count, int64_t* all_pos, double* all_val,
                int32_t* all_count, int32_t* rounds, int32_t* unresolved, double* t0, double* t1,
                void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ smallnum */
/*
 * smallnum.py:54-142 for one row-major complex128 matrix a (m x n), single-thread
 * device kernel over the hot path's small-LA code.  op: 0 svd (u m x m, s, v n x n),
 * 1 lstsq with numpy's cutoff (b [m], x [n], s [n], out_i[0] = rank; m >= n),
 * 2 eigvals (n x n; x [n], out_i[0] = converged), 3 poly_roots (a = n non-leading
 * coefficients, m = 1; x, out_i[0] = count), 4 pencil_eigenvalues (a = full
 * (r+1) x (r+1) pencil, rank; x, out_i = {rank used, ok}).  Caps: short side <= 8,
 * long side <= 32.
 */
int afft_small_la(int32_t op, int32_t m, int32_t n, const double* a, const double* b,
                  int32_t rank, double* out_u, double* out_s, double* out_v, double* out_x,
                  int32_t* out_i, void* stream);

/* ------------------------------------------------------------------ sFFT-DT1/2/3 */
/*
 * Measurement rows (oneshot.py:86-106): rows[s][bucket][3*a_m + p] = bucket values at the
 * structured shifts -a_m..2a_m-1 then the p random shifts rand_shifts[s][0..p) (device,
 * raw values as drawn by rng.choice(n, p, replace=False) with each signal's seed).
 */
int afft_bucketize_table(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld,
                         int64_t b, const int64_t* shift_table, int32_t nshift, double* out,
                         int64_t out_signal_stride, int64_t out_shift_stride,
                         int64_t out_bin_stride, void* stream);
int afft_dt_collect(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld, int64_t b,
                    int32_t a_m, int32_t p, const int64_t* rand_shifts, double* rows,
                    void* stream);

/*
 * detect_sparsity (oneshot.py:116-140) over nrows rows per signal (R measurements each):
 * sigmas [batch][nrows][a_m] (out), counts [batch][nrows] (out).
 */
int afft_dt_detect(const double* rows, int64_t batch, int64_t nrows, int32_t R, int32_t a_m,
                   int32_t k, int32_t* counts, double* sigmas, void* stream);

/* locate (oneshot.py:161-200) per row: out_pos [count][4], out_n [count] (-1 = None). */
int afft_dt_locate(const double* rows, int64_t count, int32_t R, int32_t a_m, const int32_t* a,
                   const int64_t* bucket, int32_t variant /* 1 dt1, 2 dt2, 3 dt3 */, int64_t b,
                   int64_t n, int64_t* out_pos, int32_t* out_n, void* stream);

/* estimate_values (oneshot.py:203-257) per row from candidates [count][4] (ncand each). */
int afft_dt_estimate(const double* rows, const int64_t* rand_shifts, int64_t count, int32_t a_m,
                     int32_t p, const int64_t* cands, const int32_t* ncand, int64_t b, int64_t n,
                     int64_t* out_pos, double* out_val, int32_t* out_n, void* stream);

/*
 * The per-bucket loop of sfft_dt (oneshot.py:279-288) for every row with counts > 0:
 * locate + estimate, entries to out_pos/out_val [batch][nrows][a_m], out_cnt [batch][nrows].
 * bucket_ids [batch][nrows] maps rows to bucket indices (NULL = row index); a_cap > 0
 * caps a (dsfft.py:219).
 */
int afft_dt_solve(const double* rows, const int64_t* rand_shifts, int64_t batch, int64_t nrows,
                  int32_t a_m, int32_t p, const int32_t* counts, const int64_t* bucket_ids,
                  int32_t variant, int32_t a_cap, int64_t b, int64_t n, int64_t* out_pos,
                  double* out_val, int32_t* out_cnt, void* stream);

/* Entries in row order -> all_* [batch][nrows*a_m] and the top-k truncation out_* [batch][k]. */
int afft_dt_truncate(const int64_t* pos, const double* val, const int32_t* cnt, int64_t batch,
                     int64_t nrows, int32_t a_m, int32_t k, int64_t* all_pos, double* all_val,
                     int32_t* all_count, int64_t* out_pos, double* out_val, int32_t* out_count,
                     void* stream);

/* sfft_dt (oneshot.py:266-289) over a batch: collect, detect, solve, truncate. */
size_t afft_sfft_dt_workspace_size(int64_t n, int64_t batch, int64_t b, int32_t a_m, int32_t p);
int afft_sfft_dt(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld, int64_t b,
                 int32_t a_m, int32_t p, int32_t variant, int32_t k, const int64_t* rand_shifts,
                 int64_t* out_pos, double* out_val, int32_t* out_count, int64_t* all_pos,
                 double* all_val, int32_t* all_count, int32_t* counts_out, void* workspace,
                 size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ DSFFT tree layers */

/*
 * Rows of selected buckets at arbitrary shifts (dsfft.py:118-174, 201-228):
 * rows[r][t] = bucketize(x, b, shifts[t]).values[bucket_idx[r]] for one signal, with
 * shifts sharing a coset mod n/b served by one DFT; energy [b] (may be NULL) gets
 * sum_t |bucketize(x, b, shifts[t]).values[i]|^2 for every bucket.
 */
int afft_bucketize_rows(const void* x, int dtype, int64_t n, int64_t b,
                        const int64_t* shifts /* host */, int32_t nshift,
                        const int64_t* bucket_idx, int64_t nrows, double* rows, double* energy,
                        void* stream);

/*
 * The same rows from the signal's resident spectrum Y = fft(x)/n (complex128 [n],
 * e.g. afft_bucketize with b = n, tau = 0), by the alias identity
 *   bucketize(x, b, tau)[i] = w_n^(i tau) * sum_{l < n/b} Y[i + l b] * w_(n/b)^(l tau)
 * (equal to afft_bucketize_rows up to rounding).  Rows need n/b <= 256; energy [b]
 * and values0 [b] (the tau = 0 values of every bucket, may be NULL) need n/b <= 32
 * (AFFT_EUNSUPPORTED otherwise).  Replaces dsfft.py:88-95, 159-160 at the deep layers.
 */
int afft_alias_rows(const double* spectrum, int64_t n, int64_t b, const int64_t* shifts /* host */,
                    int32_t nshift, const int64_t* bucket_idx, int64_t nrows, double* rows,
                    double* energy, double* values0, void* stream);

/*
 * Ascending indices i < b with |values[i]| > thr (dsfft.py:78, 114); with map != NULL the
 * written value is map[i].  out_count is a device int32.
 */
int afft_active_indices(const double* values, int64_t b, double thr, const int64_t* map,
                        int64_t* out_idx, int32_t* out_count, void* stream);

/* expand_layer's selective direct sums (dsfft.py:99-109) for ncand candidate buckets. */
int afft_selective_sums(const void* x, int dtype, int64_t n, int64_t b, const int64_t* cand,
                        int64_t ncand, double* out, void* stream);

/* np.median per row of `count` values: mode 0 real values, mode 1 |complex|^2. */
int afft_median(const double* values, int32_t mode, int64_t count, int64_t batch, double* out,
                void* stream);

/*
 * The whole DSFFT decode of one signal (dsfft.py:244-267 with 69-241): the layer loop
 * runs natively (one read-back per layer), every layer on the primitives above.
 * Host inputs drawn from numpy's PCG64 by the caller: the noisy search plan
 * (anchors [c], Kay weights [m-1]; dsfft.py:142-150) and, for every possible stop
 * depth d, the DT3 random shifts dt_shifts[dt_shift_off[d] .. dt_shift_off[d+1])
 * (dsfft.py:207-212).  Output: the entries dict in insertion order (host arrays,
 * out_count set even on AFFT_ENOMEM) and a trace of [kind, depth, a, b] records:
 * 0 calibrate, 1 initial (m_d), 2 expand (m_d, candidates or -1), 3 classify
 * (#single, #multi), 4 resolve (#buckets, p), 5 classify read set (R, mode).
 * full_classify = 0 lets a noisy decode classify only a probe set at the layers whose
 * entries the reference discards (dsfft.py:188-192 keeps only the last classify's
 * entries; an intermediate layer only decides whether any multi-ton remains): same
 * output, and classify records of probe layers carry #single = -1.  1 classifies every
 * active bucket at every layer (the reference's per-layer counts in the trace).
 */
typedef struct {
  double theta;          /* DsfftConfig.theta (stop rule) */
  int32_t mode;          /* 0 exact, 1 noisy */
  int32_t a_m;
  double noise_std;      /* <= 0: calibrate (noisy mode) */
  double activity_floor; /* DsfftConfig.activity_floor */
  int32_t c, m;          /* noisy search plan */
  const int64_t* anchors;
  const double* weights;
  const int64_t* dt_shifts;
  const int32_t* dt_shift_off; /* [log2(n) + 2] */
  int32_t full_classify;       /* 1: every layer classified in full (exact trace counts) */
} AfftDsfftParams;

int afft_dsfft(const void* x, int dtype, int64_t n, int32_t k, const AfftDsfftParams* params,
               int64_t* out_pos /* host */, double* out_val /* host */, int64_t capacity,
               int64_t* out_count /* host */, int32_t* trace /* host */, int32_t trace_capacity,
               int32_t* trace_len /* host */, void* stream);

/*
 * dsfft for a batch of signals (x [batch][ld], one power-of-two n) in lockstep: the
 * spectra and every full layer's active set for all signals first, then one launch
 * sequence per classify depth for every signal sitting there (rows of all their active
 * buckets in one list, classify_noisy with per-row signal ids).  params [batch] (host)
 * as for afft_dsfft.  Outputs per signal s (host): out_pos/out_val [s][capacity],
 * out_count[s], trace [s][trace_capacity][4], trace_len[s] — identical to afft_dsfft's —
 * and fallback[s] = 1 for a signal that left the common path (exact mode, calibration,
 * a selective expansion, an active set beyond the one-pass lists, a classify needing
 * the all-bucket energy pass, leftover multitons at the bottom): decode those with
 * afft_dsfft.  Replaces the reference's per-signal dsfft loop (dsfft.py:244-267) for
 * batches such as BASELINE config 4.  Synchronises.
 */
int afft_dsfft_batch(const void* x, int dtype, int64_t n, int64_t batch, int64_t ld, int32_t k,
                     const AfftDsfftParams* params /* host [batch] */, int64_t* out_pos /* host */,
                     double* out_val /* host */, int64_t capacity, int64_t* out_count /* host */,
                     int32_t* trace /* host */, int32_t trace_capacity, int32_t* trace_len /* host */,
                     int32_t* fallback /* host */, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ALIASFFT_B200_H */

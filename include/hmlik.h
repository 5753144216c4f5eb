/*
 * hmlik.h -- C-ABI of the B200-native H-matrix Gaussian log-likelihood library.
 *
 * The hot path of PAPER.md, "Likelihood Approximation
 * With Hierarchical Matrices For Large Spatial Datasets":
 *
 *   L(theta) = -n/2 log(2 pi) - 1/2 log det C(theta) - 1/2 Z^T C(theta)^{-1} Z     Eq. (1), l.52-55
 *   C(h; theta) = sigma^2 / (2^(nu-1) Gamma(nu)) (h/ell)^nu K_nu(h/ell)             Eq. (2), l.183-188
 *   L~(theta) = -n/2 log(2 pi) - sum_i log L~_ii - 1/2 v^T v,  L~ v = Z              Eq. (4), l.259-265
 *
 * with C(theta) held in H-matrix format (sec. 2.1, Definition 1, l.152-160): a
 * geometric cluster tree over the n locations, a block cluster tree split by
 * the admissibility condition, admissible blocks compressed to accuracy eps
 * (absolute, eps * sigma^2 per block in the spectral norm: Remark 2, l.166;
 * DESIGN.md reading R4) by ACA (l.147) + QR/SVD recompression (l.87),
 * an H-Cholesky factorisation with truncated low-rank updates (l.281-283),
 * log det = 2 sum log diag(L~) (l.283) and a forward solve for the quadratic
 * form (l.265).  DESIGN.md lists every reading of the paper this library takes.
 *
 * Conventions for every entry point
 *  - All floating point is IEEE fp64.  Locations are n x 2 row-major
 *    (x0, y0, x1, y1, ...).  Vectors/matrices of data (Z, xi, outputs) are
 *    column-major n x k (column j = replicate j) in the ORIGINAL location order.
 *  - A pointer argument documented "host or device" is interpreted according to
 *    the accompanying `*_on_device` flag (0 = host memory, 1 = device memory of
 *    the handle's CUDA device).  Host buffers are copied synchronously through
 *    pinned staging; device buffers are used in place on the handle's stream.
 *  - Ownership: the library never takes ownership of caller memory and never
 *    frees it.  Handles are created by hm_build / hm_tree_build and released by
 *    hm_free / hm_tree_free.
 *  - Errors: every function returns an int status (HM_OK = 0 on success, a
 *    negative HM_ERR_* code otherwise) and never aborts the process.  A
 *    human-readable message for the last error on the calling thread is
 *    available from hm_last_error().  No function falls back to a CPU path:
 *    without a usable CUDA device, GPU entry points return HM_ERR_CUDA.
 *  - Thread-safety: a handle may be used by one thread at a time.
 */
#ifndef HMLIK_H
#define HMLIK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define HM_OK               0
#define HM_ERR_ARG         -1   /* invalid argument (sizes, NaN, theta <= 0, ...)        */
#define HM_ERR_CUDA        -2   /* CUDA runtime error / no device                         */
#define HM_ERR_NOT_SPD     -3   /* Cholesky pivot <= 0 (factor not positive definite)     */
#define HM_ERR_RANK_CAP    -4   /* a truncation needed more rank than the block capacity  */
#define HM_ERR_OOM         -5   /* device or host allocation failed                        */
#define HM_ERR_STATE       -6   /* call order violated (e.g. loglik before cholesky)       */
#define HM_ERR_TOO_LARGE   -7   /* n above the dense check-path cap HM_DENSE_NMAX          */

/* theta = (sigma^2, ell, nu), all > 0 (Eq. 2; sec. 2.2 l.187).                  */
typedef struct hm_theta { double sigma2, ell, nu; } hm_theta;

/* H-matrix parameters.  eps: accuracy per low-rank block in the spectral norm
 * (Remark 2, l.166, adaptive-rank strategy; reading R4): by default
 * ABSOLUTE, eps * sigma^2 (the paper's wording; sigma^2 makes it invariant to
 * the scale of C), or relative to the block's norm when rel_eps = 1;
 * leaf: n_min (l.211); eta: admissibility parameter (reading R2); kmax: rank
 * capacity of one low-rank block, at most 240 (HM_ERR_RANK_CAP when exceeded;
 * 0 = default 160); coop_max: most CTAs cooperating on one truncation (1..32,
 * 0 = default 16; 8 when several handles share the GPU, see hm_set_exec_grid);
 * eps_chol: accuracy of every truncation inside the H-Cholesky (same meaning
 * as eps; 0 = eps).  The paper fixes the accuracies of C~ and L~ separately
 * (l.474-476, Fig. 7: 1e-3 for C~, 1e-8 for L~); Table 3 (l.483) uses one for
 * both, which is the default.  exec_ctas: CTA cap of the handle's persistent
 * executor from hm_build on (0 = all SMs; as hm_set_exec_grid), so a handle built
 * while other handles' executors run never oversubscribes the SMs.
 * adaptive_cap = 1: rank capacity per low-rank block instead of one kmax --
 * hm_build first assembles C~ with an assembly-only plan at capacity kmax, then
 * gives every block min(kmax, 1.5 rank_C~ + 8) and plans the H-Cholesky with
 * that (less device memory: blocks, H x thin temporaries, workspaces); should a
 * factor block need more, hm_cholesky grows the capacities (x2, at most 3
 * times), re-plans, re-assembles at the same theta and factors again.  The
 * capacities stay fixed for later thetas (HM_ERR_RANK_CAP as usual beyond 3
 * retries).  0 (default) = kmax for every block.                              */
typedef struct hm_params {
    double  eps;
    int32_t leaf;
    double  eta;
    int32_t kmax;
    int32_t rel_eps;
    int32_t coop_max;
    double  eps_chol;
    int32_t exec_ctas;
    int32_t adaptive_cap;
} hm_params;

typedef struct hm_handle_s* hm_handle;          /* H-matrix of C(theta) + its factor */
typedef struct hm_tree_s*   hm_tree;            /* geometry only (host)              */

/* ---- error reporting --------------------------------------------------- */
const char* hm_last_error(void);
/* Library version string. */
const char* hm_version(void);

/* ---- geometry: cluster tree + block cluster tree (host, no GPU) --------- */
/* Build the cluster tree T_I (median bisection along the longest bounding-box
 * axis, reading R1) and the block cluster tree T_{IxI} (reading R2/R3) for n
 * host locations.  Errors: HM_ERR_ARG for n < 1, leaf < 1, eta <= 0 or a
 * non-finite coordinate.                                                   */
int hm_tree_build(const double* locs_host, int64_t n, int32_t leaf, double eta, hm_tree* out);
int hm_tree_free(hm_tree t);
/* counts[0..5] = n, #clusters, #leaf clusters, depth, #leaf blocks (full I x I),
 *                #admissible leaf blocks (full I x I).                        */
int hm_tree_counts(hm_tree t, int64_t counts[6]);
/* perm[k] = original index of the k-th point in tree order (n entries).      */
int hm_tree_perm(hm_tree t, int64_t* perm_host);
/* Clusters in pre-order: 4 int64 per cluster (lo, hi, level, is_leaf).      */
int hm_tree_clusters(hm_tree t, int64_t* out_host);
/* Leaf blocks of the FULL partition of I x I, 6 int64 per block
 * (t_lo, t_hi, s_lo, s_hi, level, admissible), in recursion order.          */
int hm_tree_blocks(hm_tree t, int64_t* out_host);

/* Diagnostics (host only): build the H-Cholesky / solve plan for the tree
 * with rank capacity kmax and write it to the binary file `path` (sections
 * of int64 count + raw task structs, see tests/plan_interp.py), or, if path
 * is NULL, only fill summary[0..7] = pool doubles, #slots, #chol VM tasks,
 * #chol truncation tasks, #chol waves, #chol launches, #solve waves,
 * #solve tasks.  HM_ERR_ARG for unsupported geometry.                       */
int hm_plan_dump(hm_tree t, int32_t kmax, const char* path, double summary[8]);

/* ---- H-matrix likelihood (GPU) ------------------------------------------ */
/* hm_build(locs, theta, eps, leaf, eta): build geometry, plan the H-Cholesky,
 * allocate device storage and assemble C~(theta) (Matern blocks with device
 * K_nu, ACA + recompression of admissible blocks).  locs: n x 2, host or
 * device (locs_on_device).  stream: cudaStream_t to run on (NULL = the
 * library's own stream).  device: CUDA ordinal.                             */
int hm_build(const double* locs, int32_t locs_on_device, int64_t n,
             hm_theta theta, hm_params params, int32_t device, void* stream,
             hm_handle* out);
int hm_free(hm_handle h);

/* Re-assemble C~(theta) for a new theta on the same locations (same tree,
 * same plan).                                                                */
int hm_assemble(hm_handle h, hm_theta theta);

/* H-Cholesky C~ = L~ L~^T in place with truncated low-rank updates (every
 * truncation at the block accuracy of hm_params: eps * sigma^2 absolute, or
 * eps relative with rel_eps = 1).  HM_ERR_NOT_SPD if a pivot is not positive;
 * HM_ERR_RANK_CAP if a truncation needs more than the block's capacity.     */
int hm_cholesky(hm_handle h);

/* Log-likelihood Eq. (4) for k data vectors Z (n x k column-major, original
 * order, host or device).  out[3*j + 0..2] = (loglik, logdet, quad) of column
 * j, written to host memory.  Requires hm_cholesky first (HM_ERR_STATE).    */
int hm_loglik(hm_handle h, const double* Z, int32_t z_on_device, int32_t k, double* out_host);

/* One full evaluation per theta (Eq. 4 at each theta of a grid, an optimiser's
 * simplex, Monte-Carlo draws): for each of n_theta thetas, assemble + Cholesky
 * + loglik for the k columns of Z (n x k, host or device; device data must be
 * complete before the call).  out: n_theta x k x 3 (host), out[3k*i + 3c + ...].
 * The evaluations are co-scheduled on the handle's GPU: S executors (the handle
 * and S - 1 sibling handles on the same tree and plan, each with its own device
 * storage and stream, created on first use and kept) run concurrently from S host
 * threads, each persistent executor capped at 1/S of the SMs.  S is the value of
 * hm_set_batch_streams (default 4), reduced to what the plan's cooperative
 * truncation groups allow (each executor needs more than 4 * (largest group - 1)
 * CTAs; hm_params.coop_max = 8 allows 4), to n_theta, and to what fits in device
 * memory.  Results are bit-identical to evaluating the thetas one at a time (the
 * CTA cap never changes the arithmetic).  Failed evaluations store
 * (-inf, nan, nan) for that theta and the rest continue; the return value is the
 * first error seen (HM_OK if none).  Afterwards the handle holds no factor
 * (hm_assemble again before hm_cholesky / hm_loglik).                        */
int hm_loglik_batch(hm_handle h, const hm_theta* thetas_host, int32_t n_theta,
                    const double* Z, int32_t z_on_device, int32_t k, double* out_host);

/* Co-scheduled evaluations on DIFFERENT handles (e.g. Monte-Carlo replicates,
 * each on its own locations, sec. 4): handle i is assembled at
 * thetas[i], factored, and evaluated on its own data Zs[i] (n_i x k, host or
 * device), concurrently, one host thread per handle, the executors splitting the
 * SMs (each must keep more than 4 * (largest cooperative group - 1) CTAs, else
 * HM_ERR_ARG).  All handles on one device, none twice.  out: nh x k x 3 (host);
 * errors as in hm_loglik_batch.                                               */
int hm_loglik_multi(int32_t nh, const hm_handle* handles, const hm_theta* thetas_host,
                    const double* const* Zs, int32_t z_on_device, int32_t k, double* out_host);

/* Number of co-scheduled executors hm_loglik_batch may use (0 = default 4,
 * 1 = one evaluation at a time, at most 16).  Lowering it frees the surplus
 * sibling handles' device memory.  HM_ERR_ARG outside [0, 16].               */
int hm_set_batch_streams(hm_handle h, int32_t streams);

/* Sampler (sec. 4, l.308 "Z = L~ xi"): Z = L~ xi for k standard-normal
 * columns xi (n x k, original order, host or device); Z written in original
 * order to host or device memory.  Requires hm_cholesky first.              */
int hm_sample(hm_handle h, const double* xi, int32_t xi_on_device, int32_t k,
              double* Z, int32_t z_on_device);

/* Statistics.  st[0..11]: n, #dense blocks, #low-rank blocks, max rank C~,
 * max rank L~, bytes C~, bytes L~, compression ratio C~ (1 - bytes/8n^2),
 * #plan tasks, #plan waves, #kernel launches per Cholesky, widest Cholesky
 * truncation (sum of the actual widths of its stacked pieces).             */
int hm_stats(hm_handle h, double st[12]);

/* Timing of the last hm_assemble / hm_cholesky / hm_loglik on the device,
 * milliseconds (CUDA events on the handle's stream): ms[0..2].              */
int hm_timings(hm_handle h, double ms[3]);

/* Profiling (measurement support, bench.py).  hm_profile(h, 1) resets the
 * per-kernel accumulators and brackets every subsequent kernel launch of the
 * handle (and of its hm_loglik_batch siblings) with a CUDA event pair on its
 * stream; hm_profile(h, 0) stops recording.  Both synchronise the streams.  */
int hm_profile(hm_handle h, int32_t enable);

/* Execution mode of the planned phases (Cholesky, solve, sampler, recompression):
 * 2 (default) = one persistent kernel per phase claiming READY tasks from
 *     priority queues (k_exec_rq; priority = estimated longest path to the end),
 * 1 = one persistent kernel per phase claiming tasks in topological order and
 *     waiting for their predecessors (k_exec),
 * 0 = one launch per wave and task type (k_trunc, k_vm).
 * Same task DAG and arithmetic; a cooperative truncation sums its partials in
 * a fixed order, so all modes agree to rounding.  HM_ERR_ARG for another mode. */
int hm_set_exec_mode(hm_handle h, int32_t mode);

/* Co-scheduling: cap the persistent executor of this handle at `ctas` CTAs (one
 * per SM; 0 = all SMs).  Two handles with caps summing to the SM count, driven
 * from two host threads on two streams, run their factorisations side by side
 * (independent theta, e.g. a likelihood grid or Monte-Carlo replicates).  The
 * cap must exceed 4 * (largest cooperative truncation group - 1) of the plan,
 * else the next phase launch fails with HM_ERR_ARG.                           */
int hm_set_exec_grid(hm_handle h, int32_t ctas);

/* Diagnostics: hm_trace(h, 1, NULL) makes the persistent executor record, for
 * every task of each subsequent phase launch, (claim, dependencies-satisfied,
 * end) %globaltimer nanoseconds and (sm id | kind << 16 | CTA << 32), 4 uint64
 * per task in the phase's topological task order, followed by 64 uint64 per
 * task (randomized truncations: start and each stage boundary; else 0);
 * hm_trace(h, e, path) first
 * writes the record of the LAST executor launch to the binary file `path`
 * (if path != NULL), then sets tracing to e.                                */
int hm_trace(hm_handle h, int32_t enable, const char* path);

/* Diagnostics: checksums of the current block storage (C~ or L~): out[0] sum
 * of |entries| of dense blocks, out[1] a position-weighted sum of them, out[2]
 * sum of |entries| of the first rank(b) columns of every U_b, V_b, out[3] sum
 * of the ranks.  Copies the block storage to the host (slow; tests only).     */
int hm_checksum(hm_handle h, double out[4]);

/* Diagnostics: the matrix the handle currently holds -- C~ after hm_build /
 * hm_assemble (symmetric: its stored lower block triangle mirrored), L~ after
 * hm_cholesky (lower triangular in tree order) -- expanded to a dense n x n
 * column-major host array in the ORIGINAL point order, out[pi + pj*n] with
 * (pi, pj) = (perm[i], perm[j]) for tree positions (i, j), so that the C~ of
 * the output approximates C(theta) entry by entry and out * out^T (for L~)
 * approximates it as a whole.  8 n^2 bytes, expanded on the host (tests and
 * diagnostics only).  HM_ERR_STATE before any assembly, HM_ERR_TOO_LARGE for
 * n > HM_DENSE_NMAX.                                                         */
int hm_to_dense(hm_handle h, double* out_host);

/* Summed over the handle and its hm_loglik_batch siblings: per kernel family
 * f = 0..5 (dense Matern block generation, ACA, low-rank
 * truncation, tile VM, auxiliary gather/finish, persistent executor -- whose
 * flops/bytes are those of the truncation + VM tasks it ran): out[4f + 0] launches since
 * the last hm_profile, out[4f + 1] summed device milliseconds of those
 * launches (0 when profiling is off), out[4f + 2] algorithmic flops (kernel
 * evaluations for f = 0), out[4f + 3] algorithmic bytes, both counted by the
 * kernels themselves from their actual dimensions.       */
int hm_kernel_stats(hm_handle h, double out[24]);

/* ---- dense fp64 check path (n <= HM_DENSE_NMAX) -------------------------- */
/* Exact Eq. (1) on the GPU with dense Matern assembly, dense blocked
 * Cholesky, log det and forward solve; out[3*j+0..2] as in hm_loglik.
 * Needs 8 n^2 bytes of device memory (34 GB at n = 65,536: the configs[2]
 * reference).  HM_ERR_TOO_LARGE for n > HM_DENSE_NMAX, HM_ERR_OOM if the
 * matrix does not fit.                                                     */
#define HM_DENSE_NMAX 131072
int hm_dense_loglik(const double* locs, int32_t locs_on_device, int64_t n, hm_theta theta,
                    const double* Z, int32_t z_on_device, int32_t k,
                    int32_t device, void* stream, double* out_host);

/* Dense Matern covariance block on the GPU (test hook for the device K_nu):
 * out[i + j*ni] = C(|a_i - b_j|; theta), a: ni x 2, b: nj x 2, host arrays.  */
int hm_matern_block(const double* a_host, int64_t ni, const double* b_host, int64_t nj,
                    hm_theta theta, int32_t device, double* out_host);

#ifdef __cplusplus
}
#endif
#endif /* HMLIK_H */

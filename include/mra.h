/*
 * mra.h -- C ABI of the B200-native MRA log-likelihood library (libmra_b200.so).
 *
 * The hot path of arXiv:1905.00141: evaluating the
 * multi-resolution-approximation (MRA) Gaussian-process log-likelihood and its
 * posterior state over a multi-resolution region tree, for a fixed partition and
 * covariance parameters theta. All arithmetic is fp64 (64-bit reals).
 *
 * Conventions for every entry point
 *   - Plain pointers and sizes only. "host" pointers are ordinary CPU memory; "device"
 *     pointers are CUDA global memory on the plan's device.
 *   - Inputs are borrowed for the duration of the call (copied if kept). Outputs are
 *     caller-allocated.
 *   - No call aborts. Each returns an mra_status; mra_last_error() (thread-local) then
 *     names the argument, the region (level, index) or the CUDA call that failed.
 *   - A plan is single-entrant: one call at a time per plan.
 *   - There is no CPU fallback: every evaluation step runs in the library's sm_100a kernels;
 *     with no usable CUDA device the calls return MRA_E_CUDA.
 */
#ifndef MRA_B200_H
#define MRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mra_plan mra_plan;   /* opaque; owns host + device state of one partition */

typedef enum {
    MRA_OK = 0,
    MRA_E_ARG = 1,      /* NULL/NaN/Inf input, theta <= 0, bad size                      */
    MRA_E_CONFIG = 2,   /* J not in {2,4}, M < 1, r < 1, r_hat > 64        */
    MRA_E_STRUCT = 3,   /* degenerate bounding box, or every observation eliminated      */
    MRA_E_NUMERIC = 4,  /* a Cholesky factorization failed (not positive definite)       */
    MRA_E_CUDA = 5,     /* CUDA runtime error / no device                                  */
    MRA_E_OOM = 6,      /* device (or host) allocation failed                              */
    MRA_E_NCCL = 7      /* NCCL library missing, communicator setup or a collective failed */
} mra_status;

typedef enum {
    MRA_COV_EXP = 0,       /* sigma2 * exp(-d / rho)           ("exponential")   */
    MRA_COV_MATERN32 = 1   /* sigma2 (1 + sqrt3 d/rho) exp(-sqrt3 d/rho)  (BASELINE C2; DESIGN R3) */
} mra_cov;

/* Covariance parameters theta (PAPER.md:278 ALPHA/BETA/TAU; reading R2: tau2 is the
   nugget VARIANCE, added to the diagonal of the finest-level (observation) blocks only). */
typedef struct {
    int cov;          /* mra_cov */
    double sigma2;    /* sill, > 0 */
    double rho;       /* range, > 0 */
    double tau2;      /* nugget variance, > 0 */
} mra_theta;

/* Plan options. Zero-initialised struct or NULL = defaults. */
typedef struct {
    double offset;    /* knot margin ratio in (0, 0.5); 0 = default e/100        */
    double xscale;    /* distance scaling of x differences; 0 = 1 (DESIGN reading R4)           */
    double yscale;    /* distance scaling of y differences; 0 = 1                                */
    int device;       /* CUDA device ordinal; -1 = current device; -2 = host-only plan (structure
                         only, the paper's build_structure_only mode PAPER.md:228: info/layout work,
                         evaluations return MRA_E_CUDA)                                          */
    void* stream;     /* cudaStream_t all work is issued on (e.g. torch's current stream); NULL = legacy default */
    int rank, world;  /* subtree sharding: this process evaluates the subtrees   */
                      /* assigned to `rank` of `world`; world <= 1 = the whole tree              */
    int shard_level;  /* level whose regions are the shards; 0 = auto (first level with >= 8*world regions) */
    double mem_budget_gb; /* device memory budget for the chunked bottom pass; 0 = auto        */
    int wide;         /* grid-wide task path (leaves processed by all CTAs together):
                         0 / 1 = use it (default, M >= 2), -1 = one CTA per level-(M-1) region   */
    int host_plan;    /* 0 = build the partition on the device (bounding box, leaf keys, stable radix
                         sort by leaf: SURVEY.md NEXT-2; default), 1 = on the host (OpenMP). Both give
                         the identical plan; host-only plans (device -2) always build on the host  */
    int stream_prior; /* prior chain rows of the levels >= the chunk level:
                         0 = auto (streamed when the resident rows would take more than half the
                         budget), 1 = always streamed: computed per chunk of subtrees right before
                         that chunk's posterior pass, so device memory no longer grows with the
                         number of regions (no extra arithmetic: every region's rows are still
                         computed once); -1 = always resident. A streaming plan evaluates log L
                         (mra_loglik*, mra_optimize, sharded log L) but keeps no posterior state:
                         posterior requests and mra_predict return MRA_E_CONFIG.                */
    int theta_lanes;  /* theta-batched sweeps: 0 / 1 = one evaluation at a time;
                         k > 1 = the plan keeps k evaluation contexts (each with its own stream and
                         1/k of the memory budget, sharing the partition and task lists), and
                         mra_loglik_batch* evaluates k parameter sets concurrently, so the phases'
                         tails and small launches of one theta are filled by another's work        */
    /* --- appended in round 2 (the fields above keep their offsets) --- */
    const void* nccl_id;  /* NULL = no in-library collective (world > 1 then needs the _shard / _finish
                         pair and a caller-side reduce). Otherwise the 128-byte ncclUniqueId every rank
                         of `world` received from rank 0 (mra_nccl_unique_id): the plan creates its own
                         NCCL communicator (rank, world) on `device`, and mra_loglik / mra_loglik_dev /
                         mra_loglik_batch* / mra_optimize / mra_predict run the sharded evaluation with
                         the exchange step inside the library (PAPER.md:460-462,
                         477-479): ncclBroadcast of the above-shard prior rows from rank 0, ncclReduce
                         (sum) of the packed shard-root outputs to rank 0, rank 0 merges the levels above
                         the shard level, ncclBroadcast of log L (every rank returns it) and of the
                         above-shard posterior means; posterior outputs are completed on every rank by
                         an all-reduce. Every rank must make the same calls in the same order. With
                         world == 1 the same sharded schedule runs on one rank (a test of the path).  */
    void* (*dalloc)(size_t bytes, int device, void* stream);   /* device allocator hook (e.g. torch's
                         caching allocator); NULL = cudaMalloc. Every device buffer the plan owns or
                         uses temporarily is taken from it; returns NULL on failure (-> MRA_E_OOM)  */
    void (*dfree)(void* ptr, int device, void* stream);        /* its release; required with dalloc    */
    int graph;        /* 1 = mra_loglik_dev evaluations (log L only, one context, no communicator, profiling off) are
                         captured once as a CUDA graph and replayed: theta is read from a small device buffer the
                         call refreshes, so one graph serves every (sigma2, rho, tau2) of a covariance family; it
                         is re-captured when the family or the y pointer changes. 0 = direct launches (default). */
} mra_opts;

/* Posterior state requested from an evaluation; any pointer may be NULL. */
typedef struct {
    double* mu;       /* [n_interior * r_hat] E[eta_R | y] per pre-finest region R, level-major
                         region order, in the paper's parametrization eta_R ~ N(0, C_m(Q,Q)^{-1})
                         (PAPER.md:93-97). host pointer for mra_loglik, device for _dev        */
    double* smooth;   /* [n] E[X(s_i) | y] at each observation, ORIGINAL input order, NaN for
                         eliminated observations. host / device as above                       */
    double* region_d; /* [n_regions] per-region log-det term d_R (diagnostics/parity), host    */
    double* region_u; /* [n_regions] per-region quadratic term u_R, host                        */
    double d, u;      /* root terms: log|Sigma_MRA + tau2 I| and y^T (Sigma_MRA + tau2 I)^{-1} y */
} mra_post;

/* Build the partition, knots and observation order, upload them, and size
 * the device buffers. x, y: host arrays of n coordinates (the paper's lon, lat).
 * M >= 1 levels, J in {2,4} children per region, r >= 1 requested knots (r_hat =
 * ceil(sqrt r) * floor(r / ceil(sqrt r)) are placed; r_hat <= 64 in this build).
 * Observations located exactly at a pre-finest knot are eliminated.
 * On success *out owns the plan; release it with mra_plan_destroy. */
mra_status mra_plan_create(const double* x, const double* y, uint64_t n, int M, int J, int r,
                           const mra_opts* opts, mra_plan** out);

/* Evaluate log L = -1/2 (N log 2pi + log|Sigma_MRA + tau2 I| + y^T (Sigma_MRA + tau2 I)^{-1} y)
 * (N = retained observations) by the prior pass (top-down) and the posterior pass (bottom-up)
 * of the MRA recursion (north_star).
 *   y      : HOST array of n observed values in the ORIGINAL order given to mra_plan_create.
 *   theta  : covariance parameters.
 *   loglik : out, host scalar. With world > 1 only rank 0 receives the value (others get NaN);
 *            use the _shard / _finish pair below for the collective.
 *   post   : optional posterior state (host pointers), NULL = log L only.
 * Host<->device copies of y and of the outputs happen inside the call. */
mra_status mra_loglik(mra_plan* plan, const double* y, const mra_theta* theta, double* loglik,
                      mra_post* post);

/* Same with y (and post->mu / post->smooth) as DEVICE pointers on the plan's device. */
mra_status mra_loglik_dev(mra_plan* plan, const double* d_y, const mra_theta* theta,
                          double* loglik, mra_post* post);

/* Evaluate n_theta parameter sets on the same data (likelihood sweep, e.g. C4's 4x4 grid);
 * loglik[n_theta] host output. y is a DEVICE pointer. */
mra_status mra_loglik_batch_dev(mra_plan* plan, const double* d_y, const mra_theta* theta,
                                int n_theta, double* loglik);

/* Same sweep with y a HOST array of n values in the original input order (copied to the device once,
 * SURVEY.md §8(b) mra_loglik_batch). NaN/Inf in y -> MRA_E_ARG; the first failing theta's status is
 * returned and loglik[] holds the values evaluated before it. */
mra_status mra_loglik_batch(mra_plan* plan, const double* y, const mra_theta* theta, int n_theta,
                            double* loglik);

/* Prediction (north_star's mra_predict; the paper's "prediction" calculation mode, PAPER.md:228,
 * 494, 537): posterior mean and variance of the noise-free process X (no nugget)
 * at nq query locations, under the MRA prior, given the observations and theta of the LAST
 * evaluation on this plan -- which must have requested posterior state (post->mu or post->smooth
 * non-NULL); otherwise MRA_E_ARG. Equals kriging with Sigma_MRA (queries treated as finest-level
 * points of the leaf they fall in): mean = Sigma(q,S)(Sigma(S,S)+tau2 I)^{-1} y,
 * var = Sigma(q,q) - Sigma(q,S)(Sigma(S,S)+tau2 I)^{-1} Sigma(S,q); computed per leaf from the
 * leaf's factorization and the posterior state (mu, Ltilde^{-1}, F per region) along the ancestor
 * chain.
 *   qx, qy : host arrays of nq query coordinates (any order; need not be observations).
 *   mean, var : host outputs [nq] in the caller's order; NaN for queries outside the root domain
 *               (data bounding box with top/right pushed out 1%).
 * Not available on sharded plans (MRA_E_CONFIG). */
mra_status mra_predict(mra_plan* plan, const double* qx, const double* qy, uint64_t nq, double* mean,
                       double* var);

/* The paper's "optimization" calculation mode ("a series of likelihood
 * evaluations"): maximise log L over (sigma2, rho, tau2) for the covariance family theta->cov, by a
 * derivative-free Nelder-Mead search on the log-parameters inside [lower, upper] (host C++ logic; every
 * evaluation is one mra_loglik_dev on the device). A deterministic stand-in for the paper's BOBYQA.
 *   d_y        : DEVICE array of the n observed values (original order).
 *   theta      : in: starting point (inside the bounds); out: the best point found.
 *   lower/upper: host arrays of 3 bounds {sigma2, rho, tau2} (> 0), or NULL for (0, inf).
 *   max_evals  : evaluation budget (<= 0: 200); tol: simplex size in log-parameters (<= 0: 1e-6).
 *   best_loglik, n_evals: optional outputs. Points whose factorizations fail count as -inf. */
mra_status mra_optimize(mra_plan* plan, const double* d_y, mra_theta* theta, const double* lower,
                        const double* upper, int max_evals, double tol, double* best_loglik, int* n_evals);

/* Multi-GPU subtree sharding, one process per GPU, with the exchange done by the caller
 * (plans without opts.nccl_id; with it, mra_loglik* do all of this inside the library):
 *   mra_shard_size(plan)          -> doubles in the exchange buffer (same on every rank): per level-s
 *        region the lower triangle of its q x q augmented output, packed row by row (i(i+1)/2 + j),
 *        then the regions' d, then u, then one error count (> 0: a Cholesky failed on some rank)
 *   mra_loglik_shard(plan, d_y, theta, d_xbuf)
 *        evaluates this rank's subtrees and writes their shard-root outputs into the
 *        zero-initialised DEVICE buffer d_xbuf (slots of other ranks stay zero);
 *   <the caller sum-reduces d_xbuf to rank 0, e.g. ncclReduce / torch.distributed.reduce>
 *   mra_loglik_finish(plan, theta, d_xbuf, loglik)   (rank 0) merges the levels above the
 *        shard level and returns log L (MRA_E_NUMERIC if the reduced error count is > 0). */
uint64_t mra_shard_size(const mra_plan* plan);
mra_status mra_loglik_shard(mra_plan* plan, const double* d_y, const mra_theta* theta,
                            double* d_xbuf);
mra_status mra_loglik_finish(mra_plan* plan, const mra_theta* theta, const double* d_xbuf,
                             double* loglik);

/* Posterior state on a sharded plan (S6 for G > 1: "broadcast of above-shard mu, then
 * each GPU finishes S6 locally"):
 *   mra_loglik_shard_post(plan, d_y, theta, d_xbuf)     as mra_loglik_shard, keeping this rank's
 *        merge factors (posterior state of its subtrees);
 *   <sum-reduce d_xbuf to rank 0>
 *   mra_loglik_finish_post(plan, theta, d_xbuf, loglik, d_mutop)   (rank 0) as mra_loglik_finish, and
 *        writes the posterior means of the regions above the shard level into the DEVICE buffer
 *        d_mutop[mra_mutop_size(plan)] (whitened means, then the paper's parametrization);
 *   <broadcast d_mutop from rank 0>
 *   mra_posterior_shard(plan, d_mutop, d_mu, d_smooth)   (every rank) E[eta_R | y] for the regions above
 *        the shard level and this rank's subtrees (d_mu [n_interior * r_hat], NaN for other ranks'
 *        subtrees) and E[X(s_i) | y] for this rank's observations (d_smooth [n], original order, NaN
 *        elsewhere); DEVICE pointers, either may be NULL. */
uint64_t mra_mutop_size(const mra_plan* plan);
mra_status mra_loglik_shard_post(mra_plan* plan, const double* d_y, const mra_theta* theta, double* d_xbuf);
mra_status mra_loglik_finish_post(mra_plan* plan, const mra_theta* theta, const double* d_xbuf,
                                  double* loglik, double* d_mutop);
mra_status mra_posterior_shard(mra_plan* plan, const double* d_mutop, double* d_mu, double* d_smooth);

/* Plan statistics (the paper's build_structure_only report): any pointer may
 * be NULL. n_regions = (J^M - 1)/(J - 1), n_leaves = J^(M-1). */
mra_status mra_plan_info(const mra_plan* plan, uint64_t* n_retained, int* r_hat,
                         uint64_t* n_regions, uint64_t* n_leaves, uint64_t* n_empty_leaves,
                         uint64_t* max_leaf);

/* Device-memory layout of a plan: whether it streams its prior rows (opts.stream_prior), the
 * chunk level c and the number of level-c regions per chunk of the posterior pass, and the
 * device bytes the plan holds. Any pointer may be NULL. */
mra_status mra_plan_memory(const mra_plan* plan, int* streams_prior, int* chunk_level,
                           uint64_t* chunk_regions, uint64_t* device_bytes);

/* Copies of the plan's host-side layout: perm[n_retained] (sorted position -> original index),
 * leaf_off[n_leaves + 1] (CSR offsets of each leaf in sorted order), knots x/y
 * [n_interior * r_hat] (level-major). Any pointer may be NULL. */
mra_status mra_plan_layout(const mra_plan* plan, int64_t* perm, int64_t* leaf_off,
                           double* knots_x, double* knots_y);

/* Shard assignment of a sharded plan (world > 1): the shard level and the level-shard_level
 * region indices this rank owns (longest-processing-time assignment on the per-leaf flop model,
 * the GPU analogue of the paper's sum n_j^2 dynamic split). own may be NULL. */
mra_status mra_plan_shards(const mra_plan* plan, int* shard_level, int64_t* own, uint64_t* n_own);

/* Live kernel timing: with profiling enabled every launch is bracketed by CUDA events on the
 * plan's stream; mra_kernel_times returns the accumulated device milliseconds and launch counts
 * since the last mra_profile(plan, 1) per kernel class (host arrays of MRA_NKCLASS, either may be
 * NULL):
 *   0 prior (k_prior)   1 bottom (k_bottom: one CTA per level-(M-1) region)   2 merge (k_merge)
 *   3 other (gather, final, posterior state)   4 chain (k_wide_chain: leaf V chains)
 *   5 sigma (k_wide_sigma)   6 factor (k_wide_update / _diag / _panel_x: blocked Cholesky, X = L^{-1})
 *   7 solve (k_wide_trsm: G = X [V | y])   8 syrk+merge (k_wide_mtile: Atilde = G^T G, merge at M-1)
 *   9 covgen (k_wide_covfill: the covariance blocks of the leaf chains, written to HBM) */
#define MRA_NKCLASS 10
mra_status mra_profile(mra_plan* plan, int enable);
mra_status mra_kernel_times(const mra_plan* plan, double* ms, uint64_t* launches);

/* Number of kernel launches issued by the last evaluation call on this plan. */
uint64_t mra_last_launches(const mra_plan* plan);

void mra_plan_destroy(mra_plan* plan);

/* A fresh ncclUniqueId (128 bytes written to id_out), to be created on rank 0 and sent to every rank
 * (e.g. with torch.distributed.broadcast_object_list) before mra_plan_create with opts.nccl_id.
 * MRA_E_NCCL if no NCCL library can be loaded (libnccl.so.2, or the path in $MRA_NCCL_LIB). */
mra_status mra_nccl_unique_id(void* id_out);

/* Thread-local text of the last error ("" if none). */
const char* mra_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MRA_B200_H */

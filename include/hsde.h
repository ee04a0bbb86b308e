/*
 * hsde.h -- C ABI of libhsde.so, the B200 (sm_100a, fp64) implementation of
 * the per-iteration HSDE-ADMM hot path for chordally decomposed SDPs
 * (arXiv:1611.01828; reference package `chordalsdp`).
 *
 * The reference is pure Python; it has no FFI.  Each entry point below
 * replaces one reference function on the hot path (cited file:line, paths
 * relative to /root/reference/pkg/src/chordalsdp/).  The Python shim
 * `paper_1611_01828_b200` keeps the reference's Python signatures and calls
 * these through ctypes.
 *
 * Vectors crossing this boundary use the COMPRESSED stacked layout
 *     [ x : n_c | s : n_d | y : m | v : n_d | tau ]            (length T_c)
 * i.e. the reference layout of solver.py:119-137 with x restricted to the
 * n_c covered coordinates (clique-selected, A- or c-supported), ascending in
 * the reference's column-stacked flat order.  All pointers are HOST pointers
 * unless stated; the library copies what it needs to the device.
 *
 * Return codes: 0 OK, 1 CUDA error, 2 EigenFailure (non-finite eigenvalue,
 * symmat.py:158-163), 3 FactorizationFailure (solver.py:254-259,270-273),
 * 4 bad argument (ValueError), 5 TauZero (solver.py:410-412).
 * A handle is single-threaded; it owns one CUDA stream on one device.
 */
#ifndef HSDE_H
#define HSDE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSDE_OK 0
#define HSDE_ERR_CUDA 1
#define HSDE_ERR_EIGEN 2
#define HSDE_ERR_FACTOR 3
#define HSDE_ERR_ARG 4
#define HSDE_ERR_TAUZERO 5

/* settings flags */
#define HSDE_FLAG_EXACT_UY 1   /* uy = wy - A ua by an explicit CSR pass (solver.py:241)
                                  instead of the identity A ua = S^{-1} A t        */
#define HSDE_FLAG_NO_FACTOR 2  /* skip the Schur factorisation (residual-only handle) */
#define HSDE_FLAG_COLD_EIG 4   /* no warm start of the clique eigensolves             */
#define HSDE_FLAG_NO_SPLIT 8   /* CTA cliques: no k_cone_split fast path (Jacobi only) */
#define HSDE_FLAG_JACOBI 16    /* CTA cliques: Jacobi instead of the tridiagonal cold path */

typedef struct hsde_problem_desc {
  int64_t n;                 /* ambient matrix order (informational)              */
  int32_t m;                 /* constraints                                         */
  int32_t n_c;               /* covered coordinates                                 */
  int32_t p;                 /* cliques                                             */
  int64_t n_d;               /* sum over cliques of d_k^2                           */
  int64_t nnz;               /* nonzeros of A                                       */
  const int64_t *a_row_ptr;  /* [m+1]  CSR of A over covered columns (decompose.py:148-165) */
  const int32_t *a_col;      /* [nnz]  ascending within a row                       */
  const double *a_val;       /* [nnz]                                               */
  const double *c;           /* [n_c]  objective, ORIGINAL units                    */
  const double *b;           /* [m]    right-hand side, ORIGINAL units              */
  const int64_t *clique_offsets; /* [p+1] offsets of clique blocks in s (graphs.py:225-226) */
  const int32_t *clique_sizes;   /* [p]                                             */
  const int32_t *slot_cov;       /* [n_d] covered position of each clique slot
                                     (graphs.py:184-187 gather_index, compressed)  */
  /* ---- sharding (paper_1611_01828_b200/shard.py); zero / NULL on one GPU ---- */
  const double *cover_counts;    /* [n_c] GLOBAL cover counts D (NULL: from slot_cov) */
  const uint8_t *owned;          /* [n_c] 1 if this shard owns the coordinate (NULL: all) */
  int32_t n_sep;                 /* global separator count |S|                      */
  int32_t n_sep_local;           /* separator coordinates this shard touches        */
  const int32_t *sep_local;      /* [n_sep_local] local covered index               */
  const int32_t *sep_pos;        /* [n_sep_local] position in the global list S     */
  int32_t follower;              /* 1 on every shard but the lead (replicated y, tau
                                    are counted once, by the lead)                  */
} hsde_problem_desc;

/* Multi-GPU communicator: one shard per rank, NCCL all-reduce over NVLink.
 * The unique id comes from hsde_nccl_unique_id on rank 0, broadcast by the
 * caller (e.g. torch.distributed). */
#define HSDE_NCCL_ID_BYTES 128
typedef struct hsde_comm {
  int32_t world;
  int32_t rank;
  uint8_t nccl_id[HSDE_NCCL_ID_BYTES];
} hsde_comm;

typedef struct hsde_settings {
  double alpha;              /* over-relaxation in [1,2)        (solver.py:84)     */
  double tol;                /* termination tolerance           (solver.py:82)     */
  double infeas_tau_tol;     /*                                  (solver.py:85)    */
  double infeas_kappa_tol;   /*                                  (solver.py:86)    */
  int32_t check_interval;    /*                                  (solver.py:87)    */
  int32_t normalize;         /* scale c, b to unit norm          (solver.py:88,659-665) */
  int32_t device;            /* CUDA device ordinal                                 */
  int32_t flags;             /* HSDE_FLAG_*                                         */
} hsde_settings;

/* layout / scalar info returned by hsde_info */
typedef struct hsde_info_t {
  int64_t total;             /* T_c = n_c + 2 n_d + m + 1                           */
  int32_t n_c, m, p;
  int64_t n_d, nnz;
  double sigma_c, sigma_b;   /* normalisation scales (solver.py:659-665)            */
  double zeta_scale;         /* 1 + zeta . M^{-1} zeta           (solver.py:269)    */
  int32_t schur_diagonal;    /* S = I + A P^{-1} A' is diagonal                     */
  int32_t max_clique;
  int32_t n_shards;          /* shards held by this handle                          */
  int32_t mode;              /* 0 single GPU, 1 emulated shards (one GPU), 2 NCCL   */
  int32_t half_passes;       /* 1: A passes over mirror pairs (A_ij = A_ji columns) */
  int32_t reserved;
} hsde_info_t;

typedef struct hsde_handle hsde_t;

/* Replaces setup_cache (solver.py:248-283) + _normalization_scales
 * (:659-665) + initial_state (:366-372).  Copies the problem to the device,
 * factors S = I + A P^{-1} A' (cuSOLVER, fp64) and stores S^{-1}, solves
 * M zeta on the device.  The caller may free the desc buffers on return. */
int hsde_create(const hsde_problem_desc *desc, const hsde_settings *settings, hsde_t **out);

/* Sharded variant: `nshards` shard descriptions.  With comm
 * (world >= 1): NCCL mode, exactly one shard (this rank's).  Without
 * comm and nshards > 1: all shards on one device with device-side reductions
 * (emulation; same kernels, same three all-reduce points). */
int hsde_create_sharded(const hsde_problem_desc *descs, int32_t nshards,
                        const hsde_settings *settings, const hsde_comm *comm, hsde_t **out);
int hsde_nccl_unique_id(uint8_t *out);  /* HSDE_NCCL_ID_BYTES bytes */
int hsde_shard_total(const hsde_t *h, int32_t shard, int64_t *total);
int hsde_set_state_shard(hsde_t *h, int32_t shard, const double *u, const double *w);
int hsde_get_state_shard(hsde_t *h, int32_t shard, double *u, double *w);
void hsde_destroy(hsde_t *h);
const char *hsde_last_error(const hsde_t *h);  /* h may be NULL: last create error */
int hsde_info(const hsde_t *h, hsde_info_t *out);

/* State of the ADMM loop in the normalised problem (solver.py:358-363). */
int hsde_set_state(hsde_t *h, const double *u, const double *w);
int hsde_get_state(hsde_t *h, double *u, double *w);
/* The report's vectors (solver.py:575-585, single shard): x = u_x and y = u_y in
 * the normalised units (n_c, m; the caller unscales), and hv = H' vt with
 * vt = (u_v / sigma_c) / tau summed per covered coordinate in ascending slot order
 * (the reference's unscale + np.bincount, graphs.py:251).  Null outputs are skipped. */
int hsde_report_vectors(hsde_t *h, double tau, double *x, double *y, double *hv);
int hsde_reset_state(hsde_t *h);               /* initial_state (solver.py:366-372) */
/* Change the over-relaxation alpha of subsequent iterations (iterate takes the
 * settings per call, solver.py:375-380); rebuilds the iteration graphs. */
int hsde_set_alpha(hsde_t *h, double alpha);

/* Enqueue k iterations of `iterate` (solver.py:375-395) on the handle's stream
 * (CUDA-graph replay, no host sync).  The state before the last of the k
 * iterations is kept for the merit of hsde_check. */
int hsde_iterate(hsde_t *h, int32_t k);

/* Residual check of solve_decomposed (solver.py:721-742) on the device; one
 * host sync.  out[0..7] = pres, dres, gap, tau, kappa, merit, |b|, |c|
 * (pres/dres/gap = +inf when tau <= infeas_tau_tol, as solver.py:744-757).
 * Returns HSDE_ERR_EIGEN if any PSD projection since the last check saw a
 * non-finite eigenvalue. */
#define HSDE_CHECK_LEN 8
int hsde_check(hsde_t *h, double *out);

/* Infeasibility-certificate quantities of _try_certificates (solver.py:455-505)
 * on the unscaled iterate with the original data (solver.py:758-760).
 * out: [0] b.y  [1] c.x  [2] |A'y/by + H'v/by|  [3] min clique eig of v/by
 *      [4] |A x/(-cx)|  [5] |H x/(-cx) - s/(-cx)|  [6] min clique eig of H x/(-cx)
 * Entries of a ray whose sign test fails (b.y <= 0, resp. c.x >= 0) are NaN. */
#define HSDE_CERT_LEN 7
int hsde_certificate(hsde_t *h, double *out);

/* Unit-level entry points (compressed layout, host buffers), so the
 * reference's operator oracles can be re-pointed at the device: */
int hsde_affine_project(hsde_t *h, const double *w, double *u);        /* solver.py:296-318 */
int hsde_solve_inner(hsde_t *h, const double *w12, double *u12);       /* solver.py:286-293 */
int hsde_project_cone(hsde_t *h, const double *in, double *out);       /* solver.py:321-355 */
int hsde_residuals(hsde_t *h, const double *u, double *out3);          /* solver.py:398-429 */
int hsde_get_minv_zeta(hsde_t *h, double *out);                        /* KktCache.minv_zeta */

/* Measurement hooks (bench.py): CUDA-event timing on the handle's stream. */
int hsde_time_iterations(hsde_t *h, int32_t k, float *ms);             /* graph replay      */
/* Per-kernel profile of k iterations launched eagerly with events around every
 * kernel; names/ms arrays of length HSDE_PROFILE_SLOTS (ms summed over k). */
#define HSDE_PROFILE_SLOTS 16
int hsde_profile_iterations(hsde_t *h, int32_t k, float *ms, int32_t *launches);
const char *hsde_profile_name(int32_t slot);
int hsde_sync(hsde_t *h);
/* Eigensolver statistics of the last hot projection:
 * out[0] mean Jacobi sweeps per Jacobi-solved clique, out[1] max, out[2] mean
 * over d > 32, out[3] 1 if warm starts are enabled, out[4] / out[5] fraction of
 * the d > 32 cliques the k_cone_split fast path finished / handed to the Jacobi
 * kernel in the last hot projection, out[6] mean fixed-point iterations of the
 * finished ones, out[7..9] fraction handed over because off(B) > g / 10, r > n,
 * or the fixed point stalled, out[10] fraction finished by the fast path after
 * Jacobi sweeps refreshed the basis, out[11] fraction handed to the cold path
 * because the kept basis needed a refresh (off(B) > g / 3), out[12] fraction
 * finished by the tridiagonal cold path (any reason), out[13] fraction the
 * cold path handed to the Jacobi path (close eigenvalues). */
#define HSDE_STATS_LEN 14
int hsde_stats(hsde_t *h, double *out);
/* Diagnostics: off-diagonal norm history (relative, per sweep) of the last
 * hot projection of one clique: out[0] = 1 if warm-started, out[1..] = |off|/|A|
 * after each sweep (-1 past the last).  `clique` selects the clique traced by
 * subsequent iterations.  The diagnostics buffer exists only when the handle
 * was created with HSDE_DEBUG=1 in the environment; otherwise HSDE_ERR_ARG. */
int hsde_debug_jacobi(hsde_t *h, int32_t clique, double *out64);

/* ---- Covered layout of a reference-layout problem (host, no GPU needed) ----
 * problem.compress: the reference's DecomposedProblem keeps x over all n^2
 * coordinates (chordalsdp/decompose.py:40-79: dense c, A over n^2 columns,
 * graphs.py:228 gather_index); the device iterates on the covered ones
 * (clique-selected + support of A's columns + support of c).  build marks them
 * in a bit mask (multi-threaded) and returns their number; fill writes the
 * ascending covered ids, c on them, the rank of every column id of A (pos, the
 * compressed CSR's column indices: order-preserving) and of every gather index
 * (slot_cov).  Column ids as int32 or int64 (the other pointer null).
 * HSDE_ERR_ARG on an id outside [0, n2) or more than 2^31 - 1 covered ids. */
typedef struct hsde_cover hsde_cover_t;
int hsde_cover_build(int64_t n2, const double *c_full, const int64_t *gather_index, int64_t n_gather,
                     const int32_t *a_col32, const int64_t *a_col64, int64_t nnz, hsde_cover_t **out,
                     int64_t *n_cov);
int hsde_cover_fill(const hsde_cover_t *cv, const double *c_full, const int64_t *gather_index, int64_t n_gather,
                    const int32_t *a_col32, const int64_t *a_col64, int64_t nnz, int64_t *covered,
                    double *c_cov, int32_t *pos, int32_t *slot_cov);
void hsde_cover_destroy(hsde_cover_t *cv);

/* ---- Host decomposition (no GPU needed) ------------
 * Chordal extension + maximal cliques of one block's sparsity pattern, with
 * the reference's orderings and tie-breaking (graphs.py:73-184, 217-220):
 * maximum cardinality search, greedy minimum-degree fill when the pattern is
 * not chordal (extend != 0; else HSDE_ERR_ARG = NotChordal), elimination
 * cliques kept if maximal, cliques sorted by (min node, sorted nodes).
 * Edges (ei[k], ej[k]) are 0-based pairs; self-loops and duplicates ignored. */
typedef struct hsde_pattern hsde_pattern_t;
int hsde_pattern_decompose(int32_t n, int64_t n_edges, const int32_t *ei, const int32_t *ej,
                           int32_t extend, hsde_pattern_t **out);
int hsde_pattern_sizes(const hsde_pattern_t *p, int64_t *n_cliques, int64_t *n_nodes, int64_t *n_fill,
                       int32_t *was_chordal);
/* cliques as CSR: ptr[n_cliques + 1], nodes[n_nodes] (ascending per clique) */
int hsde_pattern_cliques(const hsde_pattern_t *p, int64_t *ptr, int32_t *nodes);
/* fill edges (a < b) in the order the elimination added them */
int hsde_pattern_fill(const hsde_pattern_t *p, int32_t *fi, int32_t *fj);
void hsde_pattern_destroy(hsde_pattern_t *p);
/* The report's pattern index (solver.py:443-452 on the compressed layout): for the
 * sorted codes gi * n + gj of the aggregate pattern plus the diagonal, the 1-based
 * block and block-local (i, j), the position of the flat id gj * n + gi in the
 * sorted `covered` (clamped) and whether it is there.  Replaces np.searchsorted and
 * friends in the report; O(nq + n_covered), host only. */
int hsde_pattern_index(const int64_t *covered, int64_t n_covered, int64_t n, const int64_t *code, int64_t nq,
                       const int64_t *starts, int32_t nblocks, int64_t *block, int64_t *li, int64_t *lj,
                       int64_t *pos_c, uint8_t *hit);

/* ---- SDPA sparse-format reader (no GPU needed) -----
 * Replaces chordalsdp/sdpa.py:94-234 parse_sdpa.  text[0..len) is the file
 * (UTF-8).  On a malformed file returns HSDE_ERR_ARG and hsde_sdpa_error()
 * gives the reference's message, its 1-based line number and whether it is a
 * DuplicateEntry (thread-local, valid until the next parse on this thread).
 * Entries come back sorted by (mat, blk, i, j): mat 0 = F0, blk/i/j 0-based,
 * i <= j (lower-triangle input normalised), explicit zeros kept. */
typedef struct hsde_sdpa hsde_sdpa_t;
int hsde_sdpa_parse(const char *text, int64_t len, hsde_sdpa_t **out);
const char *hsde_sdpa_error(int64_t *line, int32_t *duplicate);
int hsde_sdpa_sizes(const hsde_sdpa_t *p, int32_t *m, int32_t *nblocks, int64_t *n_entries);
/* block_dims[nblocks] (signed: < 0 = diagonal block), b[m], entries[n_entries] */
int hsde_sdpa_data(const hsde_sdpa_t *p, int32_t *block_dims, double *b, int32_t *mat, int32_t *blk,
                   int32_t *i, int32_t *j, double *val);
void hsde_sdpa_destroy(hsde_sdpa_t *p);

#ifdef __cplusplus
}
#endif
#endif /* HSDE_H */

/*
 * fastsum_b200.h -- C ABI of the B200 stochastic Barnes-Hut hot path.
 *
 * Every entry point replaces one call the reference package makes into its
 * numba cores or tree builder (paths relative to
 * /root/reference/pkg/src/fastsum/).  All array pointers are DEVICE pointers
 * (cudaMalloc / torch CUDA tensors), C-contiguous, FP64 unless stated; outputs
 * are caller-allocated and written in place, exactly like the reference cores.
 * `stream` is a cudaStream_t (NULL = legacy default stream); work is
 * stream-ordered and the call returns without synchronising unless noted.
 *
 * Return value: 0 = ok, 1 = invalid argument, 2 = CUDA error;
 * fsb_last_error() returns a thread-local message for the last failure.
 *
 * Kernel ids follow kernels.py:34-38 (0 coulomb, 1 winding_dipole,
 * 2 smooth_exp); rr modes follow _core.py:25-27 (0 paper_ratio,
 * 1 fixed_half, 2 disabled); precision 0 = "f64" (bitwise parity mode),
 * 1 = "f32" (FP32 terms, FP64 accumulation; outputs are float).
 */
#ifndef FASTSUM_B200_H
#define FASTSUM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fsb_tree fsb_tree; /* opaque device-resident tree */

int fsb_abi_version(void);
const char *fsb_last_error(void);

/* brute_force_batch(kid, alpha, dfloor, pts, ms, queries, out) -- _core.py:80-98.
 * pts (m,3), ms (m,c), queries (n,3); out (n,) double (precision 0) or float (1). */
int fsb_brute_force_batch(int kid, double alpha, double dfloor, int precision,
                          const double *pts, const double *ms, int64_t m, int c,
                          const double *queries, int64_t n, void *out, void *stream);

/* Ground-truth helper for large problems: FP32 terms, FP64 accumulation, out double. */
int fsb_brute_force_f32acc64(int kid, double alpha, double dfloor, const double *pts,
                             const double *ms, int64_t m, int c, const double *queries,
                             int64_t n, double *out, void *stream);

/* build_tree(sources, branching_per_dim, max_depth) -- octree.py:118-239.
 * positions (m,3), masses (m,c), weights (m,).  Synchronises `stream`. */
int fsb_build_tree(const double *positions, const double *masses, const double *weights,
                   int64_t m, int c, int branching_per_dim, int max_depth, fsb_tree **out,
                   void *stream);

/* A tree from the positional bundle of Octree.core_arrays() (octree.py:110-115),
 * i.e. what a caller of _core.*_batch passes (bbox_min is unused by every core).
 * int64 index arrays, as the reference's.  Synchronises `stream`. */
int fsb_tree_from_core_arrays(const double *diameter, const double *aggregate_mass,
                              const double *center_of_mass, const int64_t *child_start,
                              const int64_t *child_count, const int64_t *child_index,
                              const int64_t *begin, const int64_t *end, const double *points,
                              const double *masses, int64_t num_nodes, int64_t num_points,
                              int channels, fsb_tree **out, void *stream);

/* info[0..7] = num_nodes, num_points, channels, branching, max_depth, depth_levels,
 *              root child count, has_export (1 if built by fsb_build_tree). */
int fsb_tree_info(const fsb_tree *tree, int64_t *info);

/* Copy the 16 reference-layout arrays (octree.py:61-67 order, minus the two
 * scalars) into caller buffers (device or pinned host: cudaMemcpyDefault):
 * bbox_min, bbox_max, diameter, aggregate_mass, aggregate_weight,
 * center_of_mass, child_start, child_count, child_index, begin, end, depth,
 * permuted_indices, points, masses, weights.  Synchronises `stream`. */
int fsb_tree_export(const fsb_tree *tree, void *const *dst, void *stream);

int fsb_tree_free(fsb_tree *tree);

/* barnes_hut_batch(*core, kid, alpha, dfloor, queries, beta, stack_cap, out, visited)
 * -- _core.py:101-129.  qperm (optional, may be NULL): evaluation order of the
 * queries (a permutation of 0..n-1); results land at the original indices.
 * visited (optional) int64 (n,). */
int fsb_barnes_hut_batch(fsb_tree *tree, int kid, double alpha, double dfloor, int precision,
                         const double *queries, int64_t n, const int32_t *qperm, double beta,
                         void *out, int64_t *visited, void *stream);

/* The paper's GPU Barnes-Hut, not the reference's: warp voting.
 * Queries are grouped as 32 consecutive positions of `order` (NULL: 0..n-1); a
 * node is accepted for the whole group (each query adds its _node_term) when it
 * is a leaf or every query of the group sees ffr >= beta, and opened for the
 * whole group otherwise, so a group walks one preorder sequence: more accurate
 * than per-query BH at the same beta, no divergence.  visited = nodes walked
 * by the group.  FP64 matches the oracle restatement bitwise. */
int fsb_barnes_hut_vote_batch(fsb_tree *tree, int kid, double alpha, double dfloor,
                              int precision, const double *queries, int64_t n,
                              const int32_t *order, double beta, void *out, int64_t *visited,
                              void *stream);

/* stochastic_batch(*core, kid, alpha, dfloor, queries, n_samples, rr_mode, seed,
 * query_offset, out, visited, path_steps, path_count) -- _core.py:215-267.
 * RNG streams are keyed on (seed, query index + query_offset, subdomain, sample). */
int fsb_stochastic_batch(fsb_tree *tree, int kid, double alpha, double dfloor, int precision,
                         const double *queries, int64_t n, const int32_t *qperm,
                         int64_t n_samples, int rr_mode, uint64_t seed, int64_t query_offset,
                         void *out, int64_t *visited, int64_t *path_steps,
                         int64_t *path_count, void *stream);

/* stochastic_batch plus the paper's options (not the reference's):
 *  - evaluation order and shared RNG streams: queries are
 *    evaluated in `order` (a permutation, NULL = 0..n-1) and each group of
 *    2^group_log2 consecutive positions shares one stream keyed on (seed,
 *    (position + query_offset) >> group_log2, subdomain, sample), so a warp
 *    follows one sampled path.  Unbiased per query.  FSB_FLAG_SHUFFLED: the
 *    order is fsb_shuffle_order(n, seed, query_offset) (the paper shuffles the
 *    grid), computed in-kernel by the warp-uniform kernel (`order` must be
 *    NULL).  FP32 with group_log2 = 5 and query_offset % 32 == 0 runs that
 *    kernel (k_sto_warp);
 *  - FSB_FLAG_ALG2: Alg. 2 of the paper's supplemental (roulette before each
 *    swap, including the subdomain's own; unbiased; the generic per-query
 *    kernel in either precision).  Without it, the reference's walk.
 * group_log2 = 0, flags = 0 and order = NULL is fsb_stochastic_batch. */
#define FSB_FLAG_ALG2 1
#define FSB_FLAG_SHUFFLED 2
int fsb_stochastic_batch_ex(fsb_tree *tree, int kid, double alpha, double dfloor,
                            int precision, const double *queries, int64_t n,
                            const int32_t *order, int64_t n_samples, int rr_mode, uint64_t seed,
                            int64_t query_offset, int group_log2, int flags, void *out,
                            int64_t *visited, int64_t *path_steps, int64_t *path_count,
                            void *stream);

/* stochastic_moments_batch(*core, kid, alpha, dfloor, queries, n_reps, rr_mode, seed,
 * mean_out, var_out) -- _core.py:270-336.  FP64 only. */
int fsb_stochastic_moments_batch(fsb_tree *tree, int kid, double alpha, double dfloor,
                                 const double *queries, int64_t n, int64_t n_reps,
                                 int rr_mode, uint64_t seed, double *mean_out, double *var_out,
                                 void *stream);

/* telescoping_batch(*core, kid, alpha, dfloor, queries, out, visited) -- _core.py:132-156. */
int fsb_telescoping_batch(fsb_tree *tree, int kid, double alpha, double dfloor, int precision,
                          const double *queries, int64_t n, void *out, int64_t *visited,
                          void *stream);

/* Spatially coherent evaluation order for queries (3-D Morton code over the
 * query bounding box, stable): perm_out (n,) int32.  Result-invariant (F8). */
int fsb_query_order(const double *queries, int64_t n, int32_t *perm_out, void *stream);

/* Seeded evaluation order of the paper's RNG-sharing groups: perm_out (n,) int32,
 * a permutation of 0..n-1 that maps every window of 2^16 consecutive positions
 * onto itself (window w: a 4-round Feistel network keyed on (seed,
 * query_offset + w * 2^16), cycle-walked into a partial window; one kernel).
 * Window-local order lets evaluate_field_host pipeline window-aligned slabs. */
int fsb_shuffle_order(int64_t n, uint64_t seed, int64_t query_offset, int32_t *perm_out,
                      void *stream);

/* post_transform (kernels.py:110-122) applied to raw sums: smooth != 0 gives
 * -ln(raw)/alpha with (+inf, flagged) for raw <= 0; otherwise values = raw.
 * raw is float (raw_is_f32 = 1) or double; raw64 (optional) receives raw as double. */
int fsb_post_transform(const void *raw, int raw_is_f32, int64_t n, int smooth, double alpha,
                       double *values, double *raw64, uint8_t *flagged, void *stream);

/* evaluate_field (estimators.py:260-323) from HOST queries to HOST results, the
 * call a host-memory caller of the reference API makes.  The query set is split
 * into `chunks` slabs whose host->device copies, evaluation and device->host
 * copies overlap on three streams (pinned host buffers give full overlap;
 * pageable ones work but serialise the copies).  Stochastic RNG streams are keyed
 * on global query indices (query_offset + slab start), so results do not depend
 * on `chunks`.  Outputs (n,): values, raw (double; may be NULL), flagged (uint8;
 * may be NULL), visited / path_steps / path_count (int64; may be NULL); the
 * counters the method does not report are zero, visited = m for brute force
 * (FieldResult, estimators.py:45-64).  Synchronises. */
enum {
  FSB_METHOD_BRUTE_FORCE = 0,
  FSB_METHOD_BARNES_HUT = 1,
  FSB_METHOD_TELESCOPING = 2,
  FSB_METHOD_STOCHASTIC = 3
};
typedef struct fsb_eval_args {
  int method;             /* FSB_METHOD_* (EstimatorConfig.method, types.py:189-229) */
  int kid;                /* kernel id */
  double alpha, dfloor;   /* KernelSpec */
  int precision;          /* 0 f64, 1 f32 */
  double beta;            /* barnes_hut opening parameter */
  int64_t n_samples;      /* stochastic samples per subdomain */
  int rr_mode;            /* stochastic roulette mode */
  uint64_t seed;          /* stochastic seed */
  int64_t query_offset;   /* stochastic: global index of query 0 */
  int smooth;             /* post-transform: kernel is smooth_exp */
  int query_order;        /* barnes_hut: evaluate in Morton order (result-invariant) */
  const double *src_pts;  /* brute force: device sources (m,3) */
  const double *src_ms;   /* brute force: device masses (m,c) */
  int64_t m;
  int c;
  int rng_group_log2;     /* stochastic: 0 = per-query streams (reference); 5 = the
                             paper's warp-shared streams over fsb_shuffle_order */
  int bh_warp_vote;       /* barnes_hut: warp voting over the evaluation order
                             (fsb_barnes_hut_vote_batch; evaluated as one slab) */
  int path_variant;       /* stochastic: 0 = the reference's walk, 1 = Alg. 2 */
} fsb_eval_args;

int fsb_evaluate_field_host(fsb_tree *tree, const fsb_eval_args *args, const double *queries,
                            int64_t n, double *values, double *raw, uint8_t *flagged,
                            int64_t *visited, int64_t *path_steps, int64_t *path_count,
                            int chunks, void *stream);

/* error_stats + rmse (reference bench.py:66-95) on device arrays: absolute errors
 * |estimates - reference| over entries flagged in neither flags_a nor flags_b
 * (uint8, either may be NULL).  out4 = {mean, lower median, max, rmse}, count =
 * entries kept (0 -> all four NaN).  Deterministic (fixed reduction order).
 * Synchronises. */
int fsb_error_stats(const double *estimates, const double *reference, const uint8_t *flags_a,
                    const uint8_t *flags_b, int64_t n, double *out4, int64_t *count,
                    void *stream);

/* Input generation on the device, byte-identical to the reference generators
 * fed by numpy default_rng(seed) (PCG64; each thread jumps the stream to its own
 * draw).  state4 = {state_hi, state_lo, inc_hi, inc_lo} of the generator before
 * the first draw.  sample_mesh_surface (scene_io.py:112-148): cdf (num_faces,)
 * = cumsum(areas / total) / last (numpy choice's table), tri (num_faces, 3, 3)
 * vertex coordinates per face, normals (num_faces, 3) for winding_dipole masses
 * (else NULL: every mass = `mass`); outputs positions (m,3), masses (m,1|3),
 * weights (m,).  make_queries (scene_io.py:188-212): kind 0 grid3d (axes ax0,
 * ax1, ax2; r1 = len(ax1), r2 = len(ax2)), 1 slice plane (su = ax0, sv = ax1,
 * r1 = len(su); geo = origin, u_axis, v_axis), 2 random uniform (geo = low,
 * high; state4 of default_rng(spec.seed)); out (n,3).  Stream-ordered. */
int fsb_sample_mesh_surface(const double *cdf, int64_t num_faces, const double *tri,
                            const double *normals, int64_t m, const uint64_t *state4,
                            double w_each, double mass, double *positions, double *masses,
                            double *weights, void *stream);
int fsb_make_queries(int kind, int64_t n, const double *ax0, const double *ax1,
                     const double *ax2, int64_t r1, int64_t r2, const double *geo,
                     const uint64_t *state4, double *out, void *stream);

/* Text writers (host code, no GPU): the reference's field CSV
 * (scene_io.py:246-262, "index,x,y,z,value,flag" with every float as Python's
 * "{:.17g}") and points file (scene_io.py:75-80, "x y z m[ my mz]"), byte for
 * byte, rows formatted on all host threads.  queries (n,3), values (n,),
 * flagged (n,) uint8; positions (m,3), masses (m,c), c in {1, 3}. */
int fsb_write_field_csv(const char *path, int64_t n, const double *queries,
                        const double *values, const uint8_t *flagged);
int fsb_write_points_file(const char *path, int64_t m, int c, const double *positions,
                          const double *masses);

/* Self-test (synchronous, default stream): the FP64 kernels' branch-free
 * division / square root against __ddiv_rn / __dsqrt_rn on n pseudo-random
 * operand pairs.  counts4 (host) = {division fast-path cases, bit mismatches,
 * square-root fast-path cases, bit mismatches}; both mismatch counts must be 0. */
int fsb_selftest_fp64(int64_t n, uint64_t seed, unsigned long long *counts4);

/* Self-test (synchronous): the FP64 Barnes-Hut acceptance shortcut (d2 against
 * (beta dm)^2 (1 +- 2^-46), the exact _ffr(q, node) >= beta inside the band;
 * _core.py:44-52, 117) against the reference's test on n query/node pairs placed
 * within a few ulps to 1e-9 of the acceptance sphere and at random.  counts2
 * (host) = {cases, mismatches}; mismatches must be 0. */
int fsb_selftest_bh_far(int64_t n, uint64_t seed, unsigned long long *counts2);

/* Measured compute ceilings for the roofline (synchronises): out2 (host) =
 * {MUFU.RSQ ops/s, Coulomb node-term interactions/s at the packed-FP32 + MUFU
 * instruction mix with every operand on chip}. */
int fsb_micro_peaks(double *out2, void *stream);

/* Benchmark utility (no reference counterpart): hold `stream` until the host
 * writes a nonzero value to *flag (page-locked host memory) or max_cycles SM
 * cycles pass, so that work enqueued behind it runs back to back. */
int fsb_gate(const int *flag, int64_t max_cycles, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTSUM_B200_H */

/*
 * fastsum_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (FP64, scalar per query, OpenMP over queries) restatement of the
 * reference package's numeric cores, used as the parity checker for the
 * B200 kernels and as the CPU baseline ("kind": "port") in bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path never calls into this file.
 *
 * Every function cites the reference line range it restates (paths relative
 * to /root/reference/pkg/src/fastsum/).  Arithmetic is written in the same
 * association order as the reference and the file is compiled with
 * -ffp-contract=off (no FMA), so results match the numba cores bit for bit
 * for the coulomb and winding kernels (exp() comes from glibc, as numba's
 * does).  Parity of this restatement is pinned against golden vectors
 * produced by the imported reference (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DIAM_FLOOR 1e-12                     /* _core.py:29, octree.py:26 */
static const double INV_4PI = 1.0 / (4.0 * 3.141592653589793); /* kernels.py:33 */

/* ---------------------------------------------------------------- rng.py */
static const uint64_t GAMMA = 0x9E3779B97F4A7C15ull; /* rng.py:22 */
static const uint64_t MIX_M1 = 0xBF58476D1CE4E5B9ull; /* rng.py:23 */
static const uint64_t MIX_M2 = 0x94D049BB133111EBull; /* rng.py:24 */

/* rng.py:32-36 */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX_M1;
    z = (z ^ (z >> 27)) * MIX_M2;
    return z ^ (z >> 31);
}

/* rng.py:39-47 */
uint64_t or_stream_key(uint64_t seed, uint64_t qi, uint64_t sub, uint64_t sample,
                       uint64_t stream) {
    uint64_t h = mix64(seed + GAMMA);
    h = mix64(h ^ (qi + GAMMA));
    h = mix64(h ^ (sub + GAMMA));
    h = mix64(h ^ (sample + GAMMA));
    h = mix64(h ^ (stream + GAMMA));
    return h;
}

/* rng.py:50-54 */
double or_uniform_draw(uint64_t key, uint64_t counter) {
    uint64_t x = mix64(key + (counter + 1ull) * GAMMA);
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------ kernels.py */
/* contribution_rows, kernels.py:49-64 */
static inline double contrib(int kid, double alpha, double dfloor, const double *m,
                             double px, double py, double pz,
                             double qx, double qy, double qz) {
    double dx = px - qx, dy = py - qy, dz = pz - qz;
    double r = sqrt(dx * dx + dy * dy + dz * dz);
    if (r < dfloor) r = dfloor;
    if (kid == 0) return -m[0] / r;
    if (kid == 1) {
        double s = INV_4PI / (r * r * r);
        return (m[0] * dx + m[1] * dy + m[2] * dz) * s;
    }
    return m[0] * exp(-alpha * r);
}

/* ----------------------------------------------------------- tree arrays */
typedef struct {
    const double *diam, *agg_mass, *com;
    const int64_t *child_start, *child_count, *child_index, *begin, *end;
    const double *pts, *ms;
    int64_t num_nodes;
    int c;
} tree_t;

/* _ffr, _core.py:44-52 */
static inline double ffr(const tree_t *t, int64_t i, double qx, double qy, double qz) {
    double dx = qx - t->com[3 * i], dy = qy - t->com[3 * i + 1], dz = qz - t->com[3 * i + 2];
    double d = t->diam[i];
    if (d < DIAM_FLOOR) d = DIAM_FLOOR;
    return sqrt(dx * dx + dy * dy + dz * dz) / d;
}

/* rr_probability, _core.py:32-41 */
double or_rr_probability(double rp, double rc, int mode) {
    if (mode == 1) return 0.5;
    if (mode == 2) return 1.0;
    double num = rp > 1.0 ? rp : 1.0;
    double den = rc > DIAM_FLOOR ? rc : DIAM_FLOOR;
    double p = num / den;
    return p < 1.0 ? p : 1.0;
}

static inline double agg_term(const tree_t *t, int kid, double alpha, double dfloor,
                              int64_t i, double qx, double qy, double qz) {
    return contrib(kid, alpha, dfloor, t->agg_mass + (int64_t)t->c * i,
                   t->com[3 * i], t->com[3 * i + 1], t->com[3 * i + 2], qx, qy, qz);
}

/* _node_term, _core.py:55-66 */
static inline double node_term(const tree_t *t, int kid, double alpha, double dfloor,
                               int64_t i, double qx, double qy, double qz) {
    if (t->child_count[i] == 0 && t->end[i] - t->begin[i] > 1) {
        double acc = 0.0;
        for (int64_t j = t->begin[i]; j < t->end[i]; ++j)
            acc += contrib(kid, alpha, dfloor, t->ms + (int64_t)t->c * j,
                           t->pts[3 * j], t->pts[3 * j + 1], t->pts[3 * j + 2], qx, qy, qz);
        return acc;
    }
    return agg_term(t, kid, alpha, dfloor, i, qx, qy, qz);
}

/* _children_term_sum, _core.py:69-77 */
static inline double children_sum(const tree_t *t, int kid, double alpha, double dfloor,
                                  int64_t i, double qx, double qy, double qz) {
    double acc = 0.0;
    int64_t s = t->child_start[i];
    for (int64_t k = 0; k < t->child_count[i]; ++k)
        acc += node_term(t, kid, alpha, dfloor, t->child_index[s + k], qx, qy, qz);
    return acc;
}

static tree_t mk_tree(const double *diam, const double *agg_mass, const double *com,
                      const int64_t *cs, const int64_t *cc, const int64_t *ci,
                      const int64_t *b, const int64_t *e, const double *pts,
                      const double *ms, int64_t num_nodes, int c) {
    tree_t t = {diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c};
    return t;
}

/* ------------------------------------------------------------ the cores */
/* brute_force_batch, _core.py:80-98 (Kahan-compensated) */
void or_brute_force_batch(int kid, double alpha, double dfloor, const double *pts,
                          const double *ms, int64_t m, int c, const double *q,
                          int64_t n, double *out) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t qi = 0; qi < n; ++qi) {
        double qx = q[3 * qi], qy = q[3 * qi + 1], qz = q[3 * qi + 2];
        double acc = 0.0, comp = 0.0;
        for (int64_t j = 0; j < m; ++j) {
            double v = contrib(kid, alpha, dfloor, ms + (int64_t)c * j, pts[3 * j],
                               pts[3 * j + 1], pts[3 * j + 2], qx, qy, qz);
            double y = v - comp;
            double tt = acc + y;
            comp = (tt - acc) - y;
            acc = tt;
        }
        out[qi] = acc;
    }
}

/* barnes_hut_batch, _core.py:101-129 (explicit stack, children pushed reversed) */
void or_barnes_hut_batch(const double *diam, const double *agg_mass, const double *com,
                         const int64_t *cs, const int64_t *cc, const int64_t *ci,
                         const int64_t *b, const int64_t *e, const double *pts,
                         const double *ms, int64_t num_nodes, int c, int kid, double alpha,
                         double dfloor, const double *q, int64_t n, double beta,
                         int64_t stack_cap, double *out, int64_t *visited) {
    tree_t t = mk_tree(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c);
#pragma omp parallel
    {
        /* the DFS stack never holds more than num_nodes entries; callers may pass a
         * smaller (or zero) stack_cap, as the reference's signature allows */
        int64_t cap = stack_cap > num_nodes + 8 ? stack_cap : num_nodes + 8;
        int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 16)
        for (int64_t qi = 0; qi < n; ++qi) {
            double qx = q[3 * qi], qy = q[3 * qi + 1], qz = q[3 * qi + 2];
            int64_t top = 1, seen = 0;
            double acc = 0.0;
            stack[0] = 0;
            while (top > 0) {
                int64_t a = stack[--top];
                seen += 1;
                if (t.child_count[a] == 0 || ffr(&t, a, qx, qy, qz) >= beta) {
                    acc += node_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
                } else {
                    int64_t s = t.child_start[a];
                    for (int64_t k = t.child_count[a] - 1; k >= 0; --k) stack[top++] = t.child_index[s + k];
                }
            }
            out[qi] = acc;
            visited[qi] = seen;
        }
        free(stack);
    }
}

/* telescoping_batch, _core.py:132-156 */
void or_telescoping_batch(const double *diam, const double *agg_mass, const double *com,
                          const int64_t *cs, const int64_t *cc, const int64_t *ci,
                          const int64_t *b, const int64_t *e, const double *pts,
                          const double *ms, int64_t num_nodes, int c, int kid, double alpha,
                          double dfloor, const double *q, int64_t n, double *out,
                          int64_t *visited) {
    tree_t t = mk_tree(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t qi = 0; qi < n; ++qi) {
        double qx = q[3 * qi], qy = q[3 * qi + 1], qz = q[3 * qi + 2];
        double acc = node_term(&t, kid, alpha, dfloor, 0, qx, qy, qz);
        int64_t seen = 1;
        for (int64_t a = 0; a < num_nodes; ++a) {
            if (t.child_count[a] > 0) {
                double kids = children_sum(&t, kid, alpha, dfloor, a, qx, qy, qz);
                double parent = agg_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
                acc += kids - parent;
                seen += 1 + t.child_count[a];
            }
        }
        out[qi] = acc;
        visited[qi] = seen;
    }
}

/* _sample_residual, _core.py:159-212 */
static inline double sample_residual(const tree_t *t, int kid, double alpha, double dfloor,
                                     int64_t a, int64_t a_ord, int64_t count_a,
                                     double delta_a, double qx, double qy, double qz,
                                     uint64_t qi, uint64_t s, uint64_t seed, int rr_mode,
                                     int variant, int64_t *steps_out, int64_t *seen_out) {
    uint64_t key_i = or_stream_key(seed, qi, (uint64_t)a_ord, s, 0);
    uint64_t key_r = or_stream_key(seed, qi, (uint64_t)a_ord, s, 1);
    double u0 = or_uniform_draw(key_i, 0);
    int64_t j = t->begin[a] + (int64_t)(u0 * (double)count_a);
    if (j >= t->end[a]) j = t->end[a] - 1;
    int64_t node = a, steps = 0, seen = 0;
    uint64_t rctr = 0;
    double prr = 1.0, resid = 0.0;
    if (variant == 1) {
        /* the paper's Alg. 2 (supplemental pseudocode pathSampleEstimator): the
         * roulette at T_{I,k} gates the swap at T_{I,k}; seen +1 per roulette
         * test, +children per committed swap (not in the reference) */
        while (t->child_count[node] > 0) {
            int64_t child = -1, cs = t->child_start[node];
            for (int64_t k = 0; k < t->child_count[node]; ++k) {
                int64_t cc = t->child_index[cs + k];
                if (t->begin[cc] <= j && j < t->end[cc]) { child = cc; break; }
            }
            double p = or_rr_probability(ffr(t, node, qx, qy, qz), ffr(t, child, qx, qy, qz),
                                         rr_mode);
            double u = or_uniform_draw(key_r, rctr);
            rctr += 1;
            seen += 1;
            if (u >= p) break;
            double delta;
            if (node == a)
                delta = delta_a;
            else
                delta = children_sum(t, kid, alpha, dfloor, node, qx, qy, qz)
                        - agg_term(t, kid, alpha, dfloor, node, qx, qy, qz);
            seen += t->child_count[node];
            prr *= p;
            double pagg = (double)(t->end[node] - t->begin[node]) / (double)count_a;
            resid += delta / (pagg * prr);
            node = child;
            steps += 1;
        }
        *steps_out = steps;
        *seen_out = seen;
        return resid;
    }
    while (t->child_count[node] > 0) {
        int64_t child = -1, cs = t->child_start[node];
        for (int64_t k = 0; k < t->child_count[node]; ++k) {
            int64_t cc = t->child_index[cs + k];
            if (t->begin[cc] <= j && j < t->end[cc]) { child = cc; break; }
        }
        double delta;
        if (node == a)
            delta = delta_a;
        else
            delta = children_sum(t, kid, alpha, dfloor, node, qx, qy, qz)
                    - agg_term(t, kid, alpha, dfloor, node, qx, qy, qz);
        seen += t->child_count[node];
        double pagg = (double)(t->end[node] - t->begin[node]) / (double)count_a;
        resid += delta / (pagg * prr);
        double rp = ffr(t, node, qx, qy, qz);
        double rc = ffr(t, child, qx, qy, qz);
        double p = or_rr_probability(rp, rc, rr_mode);
        double u = or_uniform_draw(key_r, rctr);
        rctr += 1;
        seen += 1;
        if (u >= p) break;
        prr *= p;
        node = child;
        steps += 1;
    }
    *steps_out = steps;
    *seen_out = seen;
    return resid;
}

/* stochastic_batch, _core.py:215-267.  keys == NULL: query qi draws from the
 * streams of index qi + query_offset (the reference).  keys != NULL: from the
 * streams of index keys[qi] (the paper's shared streams: every query of a
 * group carries the group's key). */
static void stochastic_core(const double *diam, const double *agg_mass, const double *com,
                            const int64_t *cs, const int64_t *cc, const int64_t *ci,
                            const int64_t *b, const int64_t *e, const double *pts,
                            const double *ms, int64_t num_nodes, int c, int kid, double alpha,
                            double dfloor, const double *q, int64_t n, int64_t n_samples,
                            int rr_mode, uint64_t seed, int64_t query_offset,
                            const uint64_t *keys, int variant, double *out, int64_t *visited,
                            int64_t *path_steps, int64_t *path_count) {
    tree_t t = mk_tree(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c);
    int64_t root_kids = t.child_count[0];
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t qi = 0; qi < n; ++qi) {
        double qx = q[3 * qi], qy = q[3 * qi + 1], qz = q[3 * qi + 2];
        int64_t seen = 0, steps_total = 0, paths = 0;
        if (root_kids == 0) {
            out[qi] = node_term(&t, kid, alpha, dfloor, 0, qx, qy, qz);
            visited[qi] = 1;
            path_steps[qi] = 0;
            path_count[qi] = 0;
            continue;
        }
        double acc = 0.0;
        for (int64_t a_ord = 0; a_ord < root_kids; ++a_ord) {
            int64_t a = t.child_index[t.child_start[0] + a_ord];
            seen += 1;
            if (t.child_count[a] == 0) {
                acc += node_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
                continue;
            }
            double cv = agg_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
            double delta_a = children_sum(&t, kid, alpha, dfloor, a, qx, qy, qz) - cv;
            int64_t count_a = t.end[a] - t.begin[a];
            double fa = 0.0;
            for (int64_t s = 0; s < n_samples; ++s) {
                int64_t st, se;
                double resid = sample_residual(&t, kid, alpha, dfloor, a, a_ord, count_a,
                                               delta_a, qx, qy, qz,
                                               keys ? keys[qi] : (uint64_t)(qi + query_offset),
                                               (uint64_t)s, seed, rr_mode, variant, &st,
                                               &se);
                fa += resid;
                steps_total += st;
                seen += se;
                paths += 1;
            }
            acc += cv + fa / (double)n_samples;
        }
        out[qi] = acc;
        visited[qi] = seen;
        path_steps[qi] = steps_total;
        path_count[qi] = paths;
    }
}

void or_stochastic_batch(const double *diam, const double *agg_mass, const double *com,
                         const int64_t *cs, const int64_t *cc, const int64_t *ci,
                         const int64_t *b, const int64_t *e, const double *pts,
                         const double *ms, int64_t num_nodes, int c, int kid, double alpha,
                         double dfloor, const double *q, int64_t n, int64_t n_samples,
                         int rr_mode, uint64_t seed, int64_t query_offset, double *out,
                         int64_t *visited, int64_t *path_steps, int64_t *path_count) {
    stochastic_core(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c, kid, alpha,
                    dfloor, q, n, n_samples, rr_mode, seed, query_offset, NULL, 0, out, visited,
                    path_steps, path_count);
}

/* The paper's options (not in the reference): shared streams (PAPER.md:323,
 * 392) -- query qi draws from the streams of index keys[qi] (keys == NULL:
 * qi + query_offset) -- and variant 1 = Alg. 2 (roulette before each swap). */
void or_stochastic_ex_batch(const double *diam, const double *agg_mass, const double *com,
                            const int64_t *cs, const int64_t *cc, const int64_t *ci,
                            const int64_t *b, const int64_t *e, const double *pts,
                            const double *ms, int64_t num_nodes, int c, int kid, double alpha,
                            double dfloor, const double *q, int64_t n, int64_t n_samples,
                            int rr_mode, uint64_t seed, int64_t query_offset,
                            const uint64_t *keys, int variant, double *out, int64_t *visited,
                            int64_t *path_steps, int64_t *path_count) {
    stochastic_core(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c, kid, alpha,
                    dfloor, q, n, n_samples, rr_mode, seed, query_offset, keys, variant, out,
                    visited, path_steps, path_count);
}

/* Warp-voting Barnes-Hut (Alg. 1 with the acceptance test voted
 * over a group; not in the reference).  Queries are grouped as 32 consecutive
 * positions of `order`; a group walks one DFS preorder (children pushed
 * reversed, as _core.py:101-129): a node is accepted -- every query of the
 * group adds its _node_term -- when it is a leaf or every query of the group
 * sees ffr >= beta, and is opened for the whole group otherwise.  visited =
 * nodes popped by the group. */
void or_barnes_hut_vote_batch(const double *diam, const double *agg_mass, const double *com,
                              const int64_t *cs, const int64_t *cc, const int64_t *ci,
                              const int64_t *b, const int64_t *e, const double *pts,
                              const double *ms, int64_t num_nodes, int c, int kid,
                              double alpha, double dfloor, const double *q, int64_t n,
                              const int32_t *order, double beta, double *out,
                              int64_t *visited) {
    tree_t t = mk_tree(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c);
    int64_t groups = (n + 31) / 32;
#pragma omp parallel
    {
        int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * (size_t)(num_nodes + 8));
#pragma omp for schedule(dynamic, 4)
        for (int64_t g = 0; g < groups; ++g) {
            int64_t idx[32];
            double acc[32];
            int cnt = 0;
            for (int64_t p = 32 * g; p < n && p < 32 * g + 32; ++p) {
                idx[cnt] = order ? (int64_t)order[p] : p;
                acc[cnt] = 0.0;
                ++cnt;
            }
            int64_t top = 1, seen = 0;
            stack[0] = 0;
            while (top > 0) {
                int64_t a = stack[--top];
                seen += 1;
                int accept = t.child_count[a] == 0;
                if (!accept) {
                    accept = 1;
                    for (int k = 0; k < cnt && accept; ++k) {
                        const double *qq = q + 3 * idx[k];
                        accept = ffr(&t, a, qq[0], qq[1], qq[2]) >= beta;
                    }
                }
                if (accept) {
                    for (int k = 0; k < cnt; ++k) {
                        const double *qq = q + 3 * idx[k];
                        acc[k] += node_term(&t, kid, alpha, dfloor, a, qq[0], qq[1], qq[2]);
                    }
                } else {
                    int64_t s0 = t.child_start[a];
                    for (int64_t k = t.child_count[a] - 1; k >= 0; --k)
                        stack[top++] = t.child_index[s0 + k];
                }
            }
            for (int k = 0; k < cnt; ++k) {
                out[idx[k]] = acc[k];
                visited[idx[k]] = seen;
            }
        }
        free(stack);
    }
}

/* stochastic_moments_batch, _core.py:270-336 */
void or_stochastic_moments_batch(const double *diam, const double *agg_mass,
                                 const double *com, const int64_t *cs, const int64_t *cc,
                                 const int64_t *ci, const int64_t *b, const int64_t *e,
                                 const double *pts, const double *ms, int64_t num_nodes,
                                 int c, int kid, double alpha, double dfloor, const double *q,
                                 int64_t n, int64_t n_reps, int rr_mode, uint64_t seed,
                                 double *mean_out, double *var_out) {
    tree_t t = mk_tree(diam, agg_mass, com, cs, cc, ci, b, e, pts, ms, num_nodes, c);
    int64_t root_kids = t.child_count[0];
#pragma omp parallel
    {
        int64_t *sub_nodes = (int64_t *)malloc(sizeof(int64_t) * (size_t)(root_kids + 1));
        int64_t *sub_ords = (int64_t *)malloc(sizeof(int64_t) * (size_t)(root_kids + 1));
        double *sub_delta = (double *)malloc(sizeof(double) * (size_t)(root_kids + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t qi = 0; qi < n; ++qi) {
            double qx = q[3 * qi], qy = q[3 * qi + 1], qz = q[3 * qi + 2];
            if (root_kids == 0) {
                mean_out[qi] = node_term(&t, kid, alpha, dfloor, 0, qx, qy, qz);
                var_out[qi] = 0.0;
                continue;
            }
            double base = 0.0;
            int64_t n_sub = 0;
            for (int64_t a_ord = 0; a_ord < root_kids; ++a_ord) {
                int64_t a = t.child_index[t.child_start[0] + a_ord];
                if (t.child_count[a] == 0)
                    base += node_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
                else
                    n_sub += 1;
            }
            int64_t w = 0;
            for (int64_t a_ord = 0; a_ord < root_kids; ++a_ord) {
                int64_t a = t.child_index[t.child_start[0] + a_ord];
                if (t.child_count[a] == 0) continue;
                double cv = agg_term(&t, kid, alpha, dfloor, a, qx, qy, qz);
                base += cv;
                sub_nodes[w] = a;
                sub_ords[w] = a_ord;
                sub_delta[w] = children_sum(&t, kid, alpha, dfloor, a, qx, qy, qz) - cv;
                w += 1;
            }
            double acc = 0.0, acc2 = 0.0;
            for (int64_t r = 0; r < n_reps; ++r) {
                double tt = 0.0;
                for (int64_t u = 0; u < n_sub; ++u) {
                    int64_t a = sub_nodes[u], st, se;
                    tt += sample_residual(&t, kid, alpha, dfloor, a, sub_ords[u],
                                          t.end[a] - t.begin[a], sub_delta[u], qx, qy, qz,
                                          (uint64_t)qi, (uint64_t)r, seed, rr_mode, 0, &st,
                                          &se);
                }
                acc += tt;
                acc2 += tt * tt;
            }
            double mean_resid = acc / (double)n_reps;
            mean_out[qi] = base + mean_resid;
            double v = acc2 / (double)n_reps - mean_resid * mean_resid;
            var_out[qi] = v > 0.0 ? v : 0.0;
        }
        free(sub_nodes);
        free(sub_ords);
        free(sub_delta);
    }
}

/* ------------------------------------------------------------- octree.py */
/* numpy's pairwise float64 add-reduction (1-D and (n,1) axis-0 sums), used
 * by octree.py:171-173 for depth-capped leaves; pinned by tests. */
static double np_pairwise_sum(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int k = 0; k < 8; ++k) r[k] = a[k * stride];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[(i + k) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise_sum(a, n2, stride) + np_pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

double or_np_sum(const double *a, int64_t n) { return 0.0 + np_pairwise_sum(a, n, 1); }

typedef struct {
    /* growable per-node arrays (preorder) */
    int64_t n, cap;
    double *bbox_min, *side, *agg_mass, *agg_weight, *com;
    int64_t *begin, *end, *depth, *kid_first, *kid_count;
    /* children lists, appended per internal node after its subtree is built */
    int64_t *kids, nk, kcap;
} build_t;

typedef struct {
    const double *pos, *masses, *weights;
    int64_t m;
    int c, d, max_depth;
    int64_t *perm, *tmp_perm, *cid, *cnt;
    double *scratch;
    build_t B;
} ctx_t;

static void grow(ctx_t *X) {
    build_t *B = &X->B;
    if (B->n < B->cap) return;
    int64_t cap = B->cap ? 2 * B->cap : 1024;
    int c = X->c;
    B->bbox_min = realloc(B->bbox_min, sizeof(double) * 3 * cap);
    B->side = realloc(B->side, sizeof(double) * cap);
    B->agg_mass = realloc(B->agg_mass, sizeof(double) * c * cap);
    B->agg_weight = realloc(B->agg_weight, sizeof(double) * cap);
    B->com = realloc(B->com, sizeof(double) * 3 * cap);
    B->begin = realloc(B->begin, sizeof(int64_t) * cap);
    B->end = realloc(B->end, sizeof(int64_t) * cap);
    B->depth = realloc(B->depth, sizeof(int64_t) * cap);
    B->kid_first = realloc(B->kid_first, sizeof(int64_t) * cap);
    B->kid_count = realloc(B->kid_count, sizeof(int64_t) * cap);
    B->cap = cap;
}

static void push_kids(build_t *B, const int64_t *k, int64_t nk, int64_t idx) {
    if (B->nk + nk > B->kcap) {
        int64_t cap = B->kcap ? 2 * B->kcap : 1024;
        while (cap < B->nk + nk) cap *= 2;
        B->kids = realloc(B->kids, sizeof(int64_t) * cap);
        B->kcap = cap;
    }
    B->kid_first[idx] = B->nk;
    B->kid_count[idx] = nk;
    memcpy(B->kids + B->nk, k, sizeof(int64_t) * nk);
    B->nk += nk;
}

/* rec(), octree.py:148-206 */
static int64_t rec(ctx_t *X, const double cell_min[3], double cell_side, int64_t b,
                   int64_t e, int dep) {
    build_t *B = &X->B;
    grow(X);
    int64_t idx = B->n++;
    int c = X->c, d = X->d;
    for (int k = 0; k < 3; ++k) B->bbox_min[3 * idx + k] = cell_min[k];
    B->side[idx] = cell_side;
    B->begin[idx] = b;
    B->end[idx] = e;
    B->depth[idx] = dep;
    B->kid_first[idx] = 0;
    B->kid_count[idx] = 0;
    int64_t n = e - b;
    if (n == 1) { /* octree.py:161-168: verbatim copy */
        int64_t j = X->perm[b];
        for (int k = 0; k < c; ++k) B->agg_mass[(int64_t)c * idx + k] = X->masses[(int64_t)c * j + k];
        B->agg_weight[idx] = X->weights[j];
        for (int k = 0; k < 3; ++k) B->com[3 * idx + k] = X->pos[3 * j + k];
        return idx;
    }
    if (dep >= X->max_depth || cell_side == 0.0) { /* octree.py:169-176 */
        double *w = X->scratch; /* 4 * n doubles */
        double *wp = X->scratch + n;
        for (int64_t i = 0; i < n; ++i) w[i] = X->weights[X->perm[b + i]];
        double wsum = 0.0 + np_pairwise_sum(w, n, 1);
        for (int k = 0; k < c; ++k) {
            double acc;
            if (c == 1) {
                for (int64_t i = 0; i < n; ++i) wp[i] = X->masses[X->perm[b + i]];
                acc = 0.0 + np_pairwise_sum(wp, n, 1);
            } else {
                acc = 0.0;
                for (int64_t i = 0; i < n; ++i) acc = acc + X->masses[(int64_t)c * X->perm[b + i] + k];
            }
            B->agg_mass[(int64_t)c * idx + k] = acc;
        }
        B->agg_weight[idx] = wsum;
        for (int k = 0; k < 3; ++k) {
            double acc = 0.0;
            for (int64_t i = 0; i < n; ++i) acc = acc + w[i] * X->pos[3 * X->perm[b + i] + k];
            B->com[3 * idx + k] = acc / wsum;
        }
        return idx;
    }
    /* octree.py:178-187: child digits, stable sort, unique */
    double csize = cell_side / (double)d;
    int64_t nc = (int64_t)d * d * d;
    int64_t *cid = X->cid + b;
    for (int64_t i = 0; i < n; ++i) {
        const double *p = X->pos + 3 * X->perm[b + i];
        int64_t r[3];
        for (int k = 0; k < 3; ++k) {
            double f = floor((p[k] - cell_min[k]) / csize);
            int64_t v = (int64_t)f;
            if (v < 0) v = 0;
            if (v > d - 1) v = d - 1;
            r[k] = v;
        }
        cid[i] = (r[0] * d + r[1]) * d + r[2];
    }
    int64_t *cnt = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[cid[i] + 1]++;
    for (int64_t k = 0; k < nc; ++k) cnt[k + 1] += cnt[k];
    int64_t *tp = X->tmp_perm;
    int64_t *tc = X->tmp_perm + n; /* sorted cids */
    {
        int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)nc);
        memcpy(pos, cnt, sizeof(int64_t) * nc);
        for (int64_t i = 0; i < n; ++i) { /* stable counting sort */
            int64_t dst = pos[cid[i]]++;
            tp[dst] = X->perm[b + i];
            tc[dst] = cid[i];
        }
        free(pos);
    }
    memcpy(X->perm + b, tp, sizeof(int64_t) * n);
    memcpy(cid, tc, sizeof(int64_t) * n);
    int64_t *kids = (int64_t *)malloc(sizeof(int64_t) * (size_t)nc);
    int64_t nk = 0;
    for (int64_t u = 0; u < nc; ++u) { /* octree.py:189-194 */
        int64_t cb = b + cnt[u], ce = b + cnt[u + 1];
        if (ce == cb) continue;
        int64_t iz = u % d, iy = (u / d) % d, ix = u / ((int64_t)d * d);
        double cmin[3] = {cell_min[0] + (double)ix * csize, cell_min[1] + (double)iy * csize,
                          cell_min[2] + (double)iz * csize};
        kids[nk++] = rec(X, cmin, csize, cb, ce, dep + 1);
    }
    free(cnt);
    push_kids(B, kids, nk, idx);
    /* octree.py:196-205: FP64 aggregates in child order */
    double w = 0.0, wc[3] = {0.0, 0.0, 0.0};
    double msum[8];
    double *ms = c <= 8 ? msum : (double *)malloc(sizeof(double) * c);
    for (int k = 0; k < c; ++k) ms[k] = 0.0;
    for (int64_t t = 0; t < nk; ++t) {
        int64_t k2 = kids[t];
        w += B->agg_weight[k2];
        for (int k = 0; k < c; ++k) ms[k] += B->agg_mass[(int64_t)c * k2 + k];
        for (int k = 0; k < 3; ++k) wc[k] += B->agg_weight[k2] * B->com[3 * k2 + k];
    }
    for (int k = 0; k < c; ++k) B->agg_mass[(int64_t)c * idx + k] = ms[k];
    B->agg_weight[idx] = w;
    for (int k = 0; k < 3; ++k) B->com[3 * idx + k] = wc[k] / w;
    if (ms != msum) free(ms);
    free(kids);
    return idx;
}

typedef struct {
    int64_t num_nodes;
    double *bbox_min, *bbox_max, *diameter, *agg_mass, *agg_weight, *com;
    int64_t *child_start, *child_count, *child_index, *begin, *end, *depth, *perm;
} or_tree_out;

/* build_tree, octree.py:118-239.  Returns 0 on success. */
int or_build_tree(const double *pos, const double *masses, const double *weights, int64_t m,
                  int c, int d, int max_depth, or_tree_out *out) {
    if (d < 2 || max_depth < 1 || m < 1) return 1;
    ctx_t X;
    memset(&X, 0, sizeof(X));
    X.pos = pos; X.masses = masses; X.weights = weights;
    X.m = m; X.c = c; X.d = d; X.max_depth = max_depth;
    X.perm = (int64_t *)malloc(sizeof(int64_t) * m);
    X.tmp_perm = (int64_t *)malloc(sizeof(int64_t) * 2 * m);
    X.cid = (int64_t *)malloc(sizeof(int64_t) * m);
    X.scratch = (double *)malloc(sizeof(double) * 2 * m);
    for (int64_t i = 0; i < m; ++i) X.perm[i] = i;
    /* octree.py:133-136 root cube */
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) { lo[k] = pos[k]; hi[k] = pos[k]; }
    for (int64_t i = 1; i < m; ++i)
        for (int k = 0; k < 3; ++k) {
            double v = pos[3 * i + k];
            if (v < lo[k]) lo[k] = v;
            if (v > hi[k]) hi[k] = v;
        }
    double side = hi[0] - lo[0];
    for (int k = 1; k < 3; ++k) if (hi[k] - lo[k] > side) side = hi[k] - lo[k];
    double root_min[3];
    for (int k = 0; k < 3; ++k) root_min[k] = (lo[k] + hi[k]) / 2.0 - side / 2.0;
    rec(&X, root_min, side, 0, m, 0);

    build_t *B = &X.B;
    int64_t n = B->n;
    out->num_nodes = n;
    out->bbox_min = B->bbox_min;
    out->agg_mass = B->agg_mass;
    out->agg_weight = B->agg_weight;
    out->com = B->com;
    out->begin = B->begin;
    out->end = B->end;
    out->depth = B->depth;
    out->bbox_max = (double *)malloc(sizeof(double) * 3 * n);
    out->diameter = (double *)malloc(sizeof(double) * n);
    out->child_start = (int64_t *)malloc(sizeof(int64_t) * n);
    out->child_count = B->kid_count;
    out->child_index = (int64_t *)malloc(sizeof(int64_t) * (n > 1 ? n - 1 : 1));
    const double sqrt3 = sqrt(3.0);
    int64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) { /* octree.py:210-225 */
        for (int k = 0; k < 3; ++k) out->bbox_max[3 * i + k] = B->bbox_min[3 * i + k] + B->side[i];
        out->diameter[i] = B->side[i] * sqrt3;
        out->child_start[i] = acc;
        for (int64_t t = 0; t < B->kid_count[i]; ++t) out->child_index[acc + t] = B->kids[B->kid_first[i] + t];
        acc += B->kid_count[i];
    }
    out->perm = X.perm;
    free(B->side); free(B->kid_first); free(B->kids);
    free(X.tmp_perm); free(X.cid); free(X.scratch);
    return 0;
}

void or_free_tree(or_tree_out *t) {
    free(t->bbox_min); free(t->bbox_max); free(t->diameter); free(t->agg_mass);
    free(t->agg_weight); free(t->com); free(t->child_start); free(t->child_count);
    free(t->child_index); free(t->begin); free(t->end); free(t->depth); free(t->perm);
    memset(t, 0, sizeof(*t));
}

/* test helper: batch of raw stream draws */
void or_draws(uint64_t seed, uint64_t qi, uint64_t sub, uint64_t sample, uint64_t stream,
              int64_t count, double *out) {
    uint64_t key = or_stream_key(seed, qi, sub, sample, stream);
    for (int64_t i = 0; i < count; ++i) out[i] = or_uniform_draw(key, (uint64_t)i);
}

/* The warp-shared mode's evaluation order (not in the reference; restates
 * k_shuffle in csrc/fs_abi.cu): windows of 2^16 positions, each permuted by a
 * 4-round balanced Feistel network (lowbias32 rounds) keyed on (seed,
 * query_offset + window start), cycle-walked into a partial last window. */
static inline uint64_t key_fold(uint64_t h, uint64_t v) { return mix64(h ^ (v + GAMMA)); }

static inline uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    return x ^ (x >> 16);
}

static inline uint32_t feistel4(uint32_t x, int hb, const uint32_t ks[4]) {
    uint32_t mask = (1u << hb) - 1u, l = x >> hb, r = x & mask;
    for (int i = 0; i < 4; ++i) {
        uint32_t f = hash32(ks[i] ^ r) & mask, nl = r;
        r = l ^ f;
        l = nl;
    }
    return (l << hb) | r;
}

void or_shuffle_order(int64_t n, uint64_t seed, int64_t query_offset, int32_t *perm) {
    const int64_t W = (int64_t)1 << 16;
    const uint64_t h = key_fold(mix64(seed + GAMMA), 0x73687566ull);
    for (int64_t base = 0; base < n; base += W) {
        uint32_t size = (uint32_t)(n - base < W ? n - base : W);
        int hb = 1;
        while ((1u << (2 * hb)) < size) ++hb;
        uint64_t hw = key_fold(h, (uint64_t)(query_offset + base)), hw1 = key_fold(hw, 1);
        uint32_t ks[4] = {(uint32_t)hw, (uint32_t)(hw >> 32), (uint32_t)hw1, (uint32_t)(hw1 >> 32)};
        for (uint32_t i = 0; i < size; ++i) {
            uint32_t y = feistel4(i, hb, ks);
            while (y >= size) y = feistel4(y, hb, ks);
            perm[base + i] = (int32_t)(base + y);
        }
    }
}

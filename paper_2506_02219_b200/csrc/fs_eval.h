// fs_eval.h -- evaluator entry points (device pointers, stream-ordered).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fs_tree.cuh"

namespace fsb {
int brute_force(int kid, double alpha, double dfloor, bool f64, const double* pts,
                const double* ms, int64_t m, int c, const double* q, int64_t n, void* out,
                cudaStream_t s);
int brute_force_f32_acc64(int kid, double alpha, double dfloor, const double* pts,
                          const double* ms, int64_t m, int c, const double* q, int64_t n,
                          double* out, cudaStream_t s);
// vote: warp-voting BH (a warp opens a node unless all its live
// lanes accept it; groups = 32 consecutive positions of the evaluation order)
int barnes_hut(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
               int64_t n, const int32_t* qperm, double beta, void* out, int64_t* visited,
               cudaStream_t s, bool vote = false);
// share = 0: per-query RNG streams (reference); share = k > 0: the 2^k consecutive
// positions of the processing order (qperm) share one stream (paper recipe)
int stochastic(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
               int64_t n, const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed,
               int64_t query_offset, void* out, int64_t* visited, int64_t* path_steps,
               int64_t* path_count, cudaStream_t s, int share = 0, int flags = 0);
// flags of stochastic(): the paper's Alg. 2 walk; the evaluation order is
// shuffle_order(n, seed, query_offset) (qperm must be null; computed in-kernel
// by the warp-uniform kernel)
constexpr int kFlagAlg2 = 1, kFlagShuffled = 2;
int stochastic_moments(FsTree* t, int kid, double alpha, double dfloor, const double* q,
                       int64_t n, int64_t n_reps, int rr_mode, uint64_t seed, double* mean_out,
                       double* var_out, cudaStream_t s);
int telescoping(FsTree* t, int kid, double alpha, double dfloor, bool f64, const double* q,
                int64_t n, void* out, int64_t* visited, cudaStream_t s);
int stochastic_fast(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                    const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed,
                    int64_t qoff, int share, float* out, int64_t* visited, int64_t* path_steps,
                    int64_t* path_count, cudaStream_t s, bool* used, bool shuffled = false);
int stochastic64(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                 const int32_t* qperm, int n_samples, int rr_mode, uint64_t seed, int64_t qoff,
                 int share, double* out, int64_t* visited, int64_t* path_steps,
                 int64_t* path_count, cudaStream_t s, bool* used);
int barnes_hut_split(FsTree* t, int kid, double alpha, double dfloor, const double* q, int64_t n,
                     const int32_t* qperm, double beta, float* out, int64_t* visited,
                     cudaStream_t s, bool* done, bool vote = false);
int post_transform(const void* raw, int raw_f32, int64_t n, int smooth, double alpha,
                   double* values, double* raw64, uint8_t* flagged, cudaStream_t s);
}  // namespace fsb

// fs_internal.h -- host-side plumbing shared by the CUDA translation units.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "fs_tree.cuh"

namespace fsb {

void set_error(const char* fmt, ...);

// Scoped NVTX range around a C-ABI entry point (header-only NVTX3: a no-op
// unless a profiling tool is attached), so Nsight timelines and ncu's
// --nvtx-include filters see the library's calls by name.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#ifdef FSB_NO_NVTX
#define FSB_RANGE(name) ((void)0)
#else
#define FSB_RANGE(name) ::fsb::NvtxRange fsb_nvtx_range_(name)
#endif

#define FS_CK(expr)                                                                   \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      ::fsb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return 2;                                                                       \
    }                                                                                 \
  } while (0)

#define FS_TRY(expr)               \
  do {                             \
    int _rc = (expr);              \
    if (_rc != 0) return _rc;      \
  } while (0)

// Keep freed stream-ordered allocations in the device's default pool instead of
// returning them to the OS at every synchronisation (the default threshold 0
// would re-map large scratch buffers on every call).
void retain_pool_memory();

// stream-ordered scratch buffer
struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  int alloc(size_t bytes, cudaStream_t st) {
    s = st;
    retain_pool_memory();
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      set_error("cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
      p = nullptr;
      return 2;
    }
    return 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return (unsigned)g;
}

// fs_build.cu
int build_tree(FsTree** out, const double* pos, const double* masses, const double* weights,
               int64_t m, int c, int d, int max_depth, cudaStream_t s);
int tree_from_arrays(FsTree** out, const double* diameter, const double* agg_mass,
                     const double* com, const int64_t* child_start, const int64_t* child_count,
                     const int64_t* child_index, const int64_t* begin, const int64_t* end,
                     const double* points, const double* masses, int64_t n, int64_t m, int c,
                     cudaStream_t s);
int level_order(FsTree* t, const int32_t* nb, const int32_t* nd, int max_dep,
                int64_t** lstart_dev, cudaStream_t s);
int ensure_bh(FsTree* t, bool f64, cudaStream_t s);
int ensure_lo(FsTree* t, bool f64, cudaStream_t s);
int ensure_fast(FsTree* t, cudaStream_t s);
int ensure_path(FsTree* t, cudaStream_t s);
int ensure_pairs(FsTree* t, cudaStream_t s);
int ensure_cm64(FsTree* t, cudaStream_t s);
// internal children of the root (the subdomains that are sampled): every query's
// stochastic path count is n_samples times this (_core.py:215-267); read once
int internal_level1(FsTree* t, cudaStream_t s, int* out);
constexpr int64_t kShuffleWindow = 1 << 16;  // positions per shuffle window (warp-shared mode)
int shuffle_order(int64_t n, uint64_t seed, int64_t qoff, int32_t* perm, cudaStream_t s);
void free_tree(FsTree* t);

}  // namespace fsb

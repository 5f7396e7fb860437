// fs_tree.cuh -- device-resident tree handle and packed node records.
//
// Reference layout (octree.py:61-67, DFS preorder) is kept on the device for
// export and for the parity paths; the evaluators read packed records:
//   * BH (preorder, skip links):      32 B FP32 / 64 B FP64 per node
//   * level order (children contiguous): geo + mass + topo (int4) per node
#pragma once
#include <atomic>
#include <mutex>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace fsb {

struct BhRec32 {
  float4 g;  // cx, cy, cz, diam  (diam = -1 marks a multi-point leaf)
  float4 m;  // m0, m1, m2, skip (int bits); multi-point leaf: m0/m1 = begin/end bits
};
struct BhRec64 {
  double4 g;
  double4 m;  // m.w = skip (int64 bits); multi-point leaf: m.x/m.y = begin/end bits
};

struct FsTree {
  int64_t n = 0, m = 0;
  int c = 1, d = 2, max_depth = 32, d_eff = 0, num_levels = 0;
  std::vector<int64_t> level_off;  // host copy, num_levels + 1 entries (level order)
  bool owns_export = false;        // reference-layout arrays present

  // reference layout (preorder), device
  double *bbox_min = nullptr, *bbox_max = nullptr, *diameter = nullptr, *agg_mass = nullptr,
         *agg_weight = nullptr, *com = nullptr;
  int64_t *child_start = nullptr, *child_count = nullptr, *child_index = nullptr,
          *begin = nullptr, *end = nullptr, *depth = nullptr, *perm = nullptr;
  double *points = nullptr, *masses = nullptr, *weights = nullptr;

  // derived, device
  int32_t *lo2pre = nullptr, *pre2lo = nullptr, *skip = nullptr;
  int32_t* fc_lo = nullptr;  // level-order index of the first child (internal nodes)

  // packed records (built on first use)
  BhRec32* bh32 = nullptr;
  BhRec64* bh64 = nullptr;
  float4 *lo_geo32 = nullptr, *lo_mass32 = nullptr;
  double4 *lo_geo64 = nullptr, *lo_mass64 = nullptr;
  int4* lo_topo = nullptr;
  float4 *pts32a = nullptr, *pts32b = nullptr;  // permuted points {x,y,z,m0}, {m1,m2,0,0}
  double4 *pts64a = nullptr, *pts64b = nullptr;
  int root_kids = 0;  // child_count[0]
  int internal_kids = -1;  // root children with children (internal_level1), -1 = not yet read
  // Guards the lazily packed records below (ensure_*): a record pointer is
  // published only after its pack kernels have completed, so a launch on any
  // stream or host thread that obtained it through ensure_* reads finished data.
  std::recursive_mutex mu;
  std::atomic<int> bh_items_hint{0};  // load-balanced BH: items emitted by the last call

  // fast FP32 stochastic / BH path (built by ensure_fast)
  static constexpr int kMaxLevels = 256;
  bool fast_ready = false;
  bool uniform_diam = false;     // every level has one cell diameter (uniform splits)
  int first_multi_level = 1 << 30;  // shallowest level holding a multi-point leaf
  float level_diam[kMaxLevels];
  double level_diam64[kMaxLevels];  // the same, exact (FP64 queue kernel's _ffr)
  // FP64 queue kernel (ensure_cm64): {cx, cy, cz, m0} and {m1, m2} per level-order node
  double4* lo_cm64 = nullptr;
  // operand ranges of the FP64 division fast path (ensure_cm64): node coordinates
  // within 2^100, first mass channel within [2^-800, 2^800]
  bool coords_in_range = false, masses_in_range = false;
  double2* lo_m12_64 = nullptr;
  float4* lo_cm32 = nullptr;     // {cx, cy, cz, m0} per level-order node
  float2* lo_m12_32 = nullptr;   // {m1, m2} (winding)
  int32_t* lo_begin = nullptr;   // point-range begin per level-order node
  // Coulomb records of node pairs (2i, 2i+1) interleaved for packed FP32 math:
  // {x0, x1, y0, y1}, {z0, z1, -m0, -m1} (ensure_pairs)
  float4* lo_cmp = nullptr;
  // per (permuted) point: rank of its ancestor among its siblings at levels
  // 1..path_levels, path_bits bits per level (child pick without begins)
  uint64_t* pt_path = nullptr;
  int path_bits = 0, path_levels = 0;
  int max_children = 0;  // (ensure_path)
};

}  // namespace fsb

// fs_io.cu -- native text writers for field results and point sets (host code).
//
// The reference formats every number with Python's "{:.17g}" in a Python loop
// (scene_io.py:75-80 points files, :246-262 the field CSV): ~3 us per row, i.e.
// seconds for the 10^6-query C4 plane and tens of seconds for the 16.8 M-query C3
// grid, next to a sub-millisecond evaluation.  These writers produce the same
// bytes (C's %.17g and Python's .17g are both correctly rounded, with the same
// exponent form; non-finite values are spelled as Python spells them), row
// blocks formatted by all host threads into private buffers and written in
// order.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fastsum_b200.h"
#include "fs_internal.h"

namespace fsb {
namespace {

// "{:.17g}" of Python (float.__format__)
inline int fmt17(char* dst, double v) {
  if (std::isnan(v)) {
    std::memcpy(dst, "nan", 3);
    return 3;
  }
  if (std::isinf(v)) {
    if (v > 0) {
      std::memcpy(dst, "inf", 3);
      return 3;
    }
    std::memcpy(dst, "-inf", 4);
    return 4;
  }
  return std::snprintf(dst, 32, "%.17g", v);
}

inline int fmt_i64(char* dst, int64_t v) { return std::snprintf(dst, 24, "%lld", (long long)v); }

// Formats rows [0, n) with row(i, buffer) -> bytes written (at most max_row) on
// all host threads, then writes the blocks to `path` in order.
template <class Row>
int write_rows(const char* path, const char* header, int64_t n, int max_row, Row row) {
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    set_error("cannot open %s for writing", path);
    return 1;
  }
  if (header) std::fputs(header, f);
  const int64_t block = 1 << 16;
  const int64_t nblocks = (n + block - 1) / block;
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nthreads = std::max<int64_t>(1, std::min<int64_t>(hw, nblocks));
  // process in rounds of nthreads blocks: bounded memory (nthreads x 64 Ki rows)
  std::vector<std::string> bufs((size_t)nthreads);
  int rc = 0;
  for (int64_t b0 = 0; b0 < nblocks && rc == 0; b0 += nthreads) {
    const int64_t nb = std::min<int64_t>(nthreads, nblocks - b0);
    auto work = [&](int64_t t) {
      const int64_t lo = (b0 + t) * block, hi = std::min(n, lo + block);
      std::string& s = bufs[(size_t)t];
      s.resize((size_t)((hi - lo) * max_row));
      char* p = &s[0];
      for (int64_t i = lo; i < hi; ++i) p += row(i, p);
      s.resize((size_t)(p - s.data()));
    };
    std::vector<std::thread> th;
    for (int64_t t = 1; t < nb; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int64_t t = 0; t < nb; ++t)
      if (std::fwrite(bufs[(size_t)t].data(), 1, bufs[(size_t)t].size(), f) !=
          bufs[(size_t)t].size()) {
        set_error("short write to %s", path);
        rc = 1;
        break;
      }
  }
  if (std::fclose(f) != 0 && rc == 0) {
    set_error("cannot close %s", path);
    rc = 1;
  }
  return rc;
}

}  // namespace
}  // namespace fsb

// scene_io.py:246-262: "index,x,y,z,value,flag" rows
extern "C" int fsb_write_field_csv(const char* path, int64_t n, const double* queries,
                                   const double* values, const uint8_t* flagged) {
  if (!path || n < 0 || (n > 0 && (!queries || !values || !flagged))) {
    fsb::set_error("fsb_write_field_csv: null argument");
    return 1;
  }
  return fsb::write_rows(path, "index,x,y,z,value,flag\n", n, 24 + 4 * 26 + 4,
                         [&](int64_t i, char* p) {
                           char* s = p;
                           s += fsb::fmt_i64(s, i);
                           for (int k = 0; k < 3; ++k) {
                             *s++ = ',';
                             s += fsb::fmt17(s, queries[3 * i + k]);
                           }
                           *s++ = ',';
                           s += fsb::fmt17(s, values[i]);
                           *s++ = ',';
                           *s++ = flagged[i] ? '1' : '0';
                           *s++ = '\n';
                           return (int)(s - p);
                         });
}

// scene_io.py:75-80: "x y z m[ my mz]" rows
extern "C" int fsb_write_points_file(const char* path, int64_t m, int c, const double* positions,
                                     const double* masses) {
  if (!path || m < 0 || c < 1 || c > 3 || (m > 0 && (!positions || !masses))) {
    fsb::set_error("fsb_write_points_file: bad argument");
    return 1;
  }
  return fsb::write_rows(path, nullptr, m, 6 * 26 + 8, [&](int64_t i, char* p) {
    char* s = p;
    for (int k = 0; k < 3 + c; ++k) {
      if (k) *s++ = ' ';
      s += fsb::fmt17(s, k < 3 ? positions[3 * i + k] : masses[(int64_t)c * i + (k - 3)]);
    }
    *s++ = '\n';
    return (int)(s - p);
  });
}

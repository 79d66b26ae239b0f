// Host-side text formatting for the output writers (write_vtk ASCII with
// 17 significant digits, io_vtk.py:22-82).  The reference formats every value with Python's
// f"{x:.17g}" one at a time; at config 3 that is ~31M values and minutes of interpreter
// time per VTK step.  Here the same correctly rounded %.17g text is produced by snprintf on
// all host cores, row blocks in parallel.  No device code.

#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/b200fem.h"

namespace {

// Python's format(x, '.17g') == C's %.17g for finite values (both correctly rounded, same
// exponent style); inf / nan are spelled the Python way (no sign on nan).
inline int fmt_g17(char *dst, double x) {
  if (std::isnan(x)) return (int)(memcpy(dst, "nan", 3), 3);
  if (std::isinf(x)) return x > 0 ? (int)(memcpy(dst, "inf", 3), 3) : (int)(memcpy(dst, "-inf", 4), 4);
  return snprintf(dst, 32, "%.17g", x);
}

inline int fmt_i64(char *dst, long long v) { return snprintf(dst, 24, "%lld", v); }

// Format rows [r0, r1) into buf; returns bytes.  prefix >= 0 -> "prefix " before each row.
template <class T>
std::vector<char> format_block(const T *v, int64_t r0, int64_t r1, int cols, long long prefix) {
  std::vector<char> out((size_t)(r1 - r0) * ((size_t)cols * 25 + 24) + 1);
  char *p = out.data();
  for (int64_t r = r0; r < r1; ++r) {
    if (prefix >= 0) {
      p += fmt_i64(p, prefix);
      *p++ = ' ';
    }
    for (int c = 0; c < cols; ++c) {
      if (c) *p++ = ' ';
      if constexpr (sizeof(T) == 8 && std::is_floating_point<T>::value) p += fmt_g17(p, (double)v[r * cols + c]);
      else p += fmt_i64(p, (long long)v[r * cols + c]);
    }
    *p++ = '\n';
  }
  out.resize(p - out.data());
  return out;
}

template <class T>
int64_t format_rows(const T *v, int64_t rows, int32_t cols, long long prefix, char *out, int64_t cap) {
  if (rows < 0 || cols <= 0 || (rows && !v)) return -1;
  int nt = (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min<int>(nt, (int)((rows + 4095) / 4096)));
  std::vector<std::vector<char>> parts(nt);
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
    th.emplace_back([&, t, r0, r1] { parts[t] = format_block<T>(v, r0, r1, cols, prefix); });
  }
  for (auto &x : th) x.join();
  int64_t total = 0;
  for (auto &pp : parts) total += (int64_t)pp.size();
  if (!out || cap < total) return -total;  // caller retries with a buffer this large
  for (auto &pp : parts) {
    memcpy(out, pp.data(), pp.size());
    out += pp.size();
  }
  return total;
}

}  // namespace

extern "C" {

int64_t b200fem_format_f64_rows(const double *v, int64_t rows, int32_t cols, char *out, int64_t cap) {
  return format_rows<double>(v, rows, cols, -1, out, cap);
}

int64_t b200fem_format_i64_rows(const int64_t *v, int64_t rows, int32_t cols, int64_t prefix, char *out,
                                int64_t cap) {
  return format_rows<int64_t>(v, rows, cols, (long long)prefix, out, cap);
}

}  // extern "C"

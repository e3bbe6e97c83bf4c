// CPU oracle, C++ part — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the plain definition of
// the k-th order statistic as the paper's CPU comparison computes it, for bench.py's cpu_baseline
// (single-core std::nth_element = the paper's CPU quickselect row, and
// std::sort) and for the pins in tests/test_oracle_pins.py.  x_(k) = the k-th element (1-based) of
// x sorted ascending.  Nothing here is shared with or called by libcpsel.so.
#include <algorithm>
#include <cstdint>
#include <vector>

namespace {
template <typename T> T nth(const T* x, uint64_t n, uint64_t k) {
  std::vector<T> c(x, x + n);                       // the sample is immutable: work on a copy
  std::nth_element(c.begin(), c.begin() + (k - 1), c.end());
  return c[k - 1];
}
template <typename T> T by_sort(const T* x, uint64_t n, uint64_t k) {
  std::vector<T> c(x, x + n);
  std::sort(c.begin(), c.end());
  return c[k - 1];
}
}  // namespace

extern "C" {
// k in [1, n], x finite (the callers check); the value is returned as a double (exact for both)
double oracle_nth_element_f32(const float* x, uint64_t n, uint64_t k) { return nth(x, n, k); }
double oracle_nth_element_f64(const double* x, uint64_t n, uint64_t k) { return nth(x, n, k); }
double oracle_sort_select_f32(const float* x, uint64_t n, uint64_t k) { return by_sort(x, n, k); }
double oracle_sort_select_f64(const double* x, uint64_t n, uint64_t k) { return by_sort(x, n, k); }
}

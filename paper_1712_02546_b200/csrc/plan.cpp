// plan.cpp — partition map of the method (a1): Eq. 1 + exact-integer largest remainder.
//
// P:L145-153 (§4.1.1): each device times a probe convolution (t_i); the workload
// (number of kernels) of device i is proportional to w_i = (max t / t_i) / sum_j (max t / t_j)
// (Eq. 1).  The paper gives no integer rule; we apportion by largest remainder
// over exact integers (reading R11) so that the map is
// bit-identical on every rank and independent of floating-point summation order.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"

extern "C" int cp_eq1_weights(const double* t, int32_t n, double* w) {
  if (!t || !w) CP_FAIL(CP_ERR_ARG, "cp_eq1_weights: null pointer");
  if (n < 1 || n > CP_MAX_RANKS) CP_FAIL(CP_ERR_CONFIG, "cp_eq1_weights: n_ranks out of range");
  double tmax = 0;
  for (int i = 0; i < n; ++i) {
    if (!(t[i] > 0) || !std::isfinite(t[i]))
      CP_FAIL(CP_ERR_DATA, "cp_eq1_weights: nonpositive or non-finite time at rank " + std::to_string(i));
    tmax = std::max(tmax, t[i]);
  }
  double den = 0;
  for (int j = 0; j < n; ++j) den += tmax / t[j];
  for (int i = 0; i < n; ++i) w[i] = (tmax / t[i]) / den;
  return CP_OK;
}

extern "C" int cp_partition_plan(const double* t, int32_t n, int32_t num_k, int32_t align,
                                 cp_partition* out) {
  if (!t || !out) CP_FAIL(CP_ERR_ARG, "cp_partition_plan: null pointer");
  if (n < 1 || n > CP_MAX_RANKS) CP_FAIL(CP_ERR_CONFIG, "cp_partition_plan: n_ranks out of range");
  if (align < 1) CP_FAIL(CP_ERR_CONFIG, "cp_partition_plan: align < 1");
  if (num_k < 0) CP_FAIL(CP_ERR_ARG, "cp_partition_plan: num_k < 0");
  double tmax = 0;
  for (int i = 0; i < n; ++i) {
    if (!(t[i] > 0) || !std::isfinite(t[i]))
      CP_FAIL(CP_ERR_DATA, "cp_partition_plan: nonpositive or non-finite time at rank " + std::to_string(i));
    tmax = std::max(tmax, t[i]);
  }
  // quantised relative throughputs, q_i >= 2^20
  std::vector<__int128> q(n);
  __int128 sq = 0;
  for (int i = 0; i < n; ++i) {
    const double ratio = tmax / t[i];
    if (ratio > 1e12) CP_FAIL(CP_ERR_DATA, "cp_partition_plan: throughput ratio above 1e12");
    q[i] = (__int128)std::llround(1048576.0 * ratio);
    sq += q[i];
  }
  std::vector<int> cnt(n);
  std::vector<__int128> rem(n);
  int given = 0;
  for (int i = 0; i < n; ++i) {
    const __int128 num = (__int128)num_k * q[i];
    cnt[i] = (int)(num / sq);
    rem[i] = num % sq;
    given += cnt[i];
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rem[a] > rem[b]; });
  for (int j = 0; j < num_k - given; ++j) cnt[order[j]] += 1;  // leftover < n by construction
  *out = cp_partition{};
  out->n_ranks = n;
  out->num_k = num_k;
  int b = 0;
  for (int i = 0; i < n; ++i) {
    out->k_begin[i] = b;
    out->k_count[i] = cnt[i];
    out->k_width[i] = (cnt[i] + align - 1) / align * align;
    b += cnt[i];
  }
  return CP_OK;
}

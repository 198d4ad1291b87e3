// search.cuh -- per-instance partition search, shared by the batch search kernel, the fused
// predict->search kernel and the simulator kernel.
//
// Restates optimize_partition (optimizer.hpp:62-115) as a static, rank-ordered scan over the
// 111 (entry, permutation) candidates of candidates_gen.cuh:
//   * objective = FP64 left-to-right sum in job order (optimizer.hpp:78-87). This TU family is
//     compiled with --fmad=false, so every '+' is one IEEE DADD, bit-exact with the reference;
//   * an assignment is valid iff every used speed is > 0 (optimizer.hpp:82); invalid speeds are
//     poisoned to -inf so they can never win (NaN also fails '> 0');
//   * ties: candidates are visited in OptKey rank order (total_gpc, shape, placement;
//     optimizer.hpp:46-51) and only a strictly greater objective replaces the incumbent.
#pragma once
#include <cstdint>

#include "candidates_gen.cuh"

namespace miso_b200 {

constexpr uint8_t kCandInfeasible = 0xFF;
constexpr uint8_t kCandBadM = 0xFE;

__device__ __forceinline__ double poison(double x) {
  return x > 0.0 ? x : __longlong_as_double(0xFFF0000000000000ll);  // -inf
}

template <int M>
__device__ __forceinline__ int search_fixed(const double (&v)[M][5], double& best, uint64_t en0,
                                            uint64_t en1) {
  if constexpr (M == 1) return search_m1(v, best, en0, en1);
  else if constexpr (M == 2) return search_m2(v, best, en0, en1);
  else if constexpr (M == 3) return search_m3(v, best, en0, en1);
  else if constexpr (M == 4) return search_m4(v, best, en0, en1);
  else if constexpr (M == 5) return search_m5(v, best, en0, en1);
  else if constexpr (M == 6) return search_m6(v, best, en0, en1);
  else return search_m7(v, best, en0, en1);
}

// Scores one instance whose m x 5 speed rows start at `row` (any address space).
// Returns the candidate id or kCandInfeasible; *obj receives the objective (0 if none).
template <int M, class Ptr>
__device__ __forceinline__ uint8_t search_rows(Ptr row, uint64_t en0, uint64_t en1, double* obj) {
  double v[M][5];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int k = 0; k < 5; ++k) v[i][k] = poison(row[i * 5 + k]);
  double best = __longlong_as_double(0xFFF0000000000000ll);
  int c = search_fixed<M>(v, best, en0, en1);
  *obj = c < 0 ? 0.0 : best;
  return c < 0 ? kCandInfeasible : static_cast<uint8_t>(c);
}

template <class Ptr>
__device__ __forceinline__ uint8_t search_any(Ptr row, int m, uint64_t en0, uint64_t en1,
                                              double* obj) {
  switch (m) {
    case 1: return search_rows<1>(row, en0, en1, obj);
    case 2: return search_rows<2>(row, en0, en1, obj);
    case 3: return search_rows<3>(row, en0, en1, obj);
    case 4: return search_rows<4>(row, en0, en1, obj);
    case 5: return search_rows<5>(row, en0, en1, obj);
    case 6: return search_rows<6>(row, en0, en1, obj);
    case 7: return search_rows<7>(row, en0, en1, obj);
    default: *obj = 0.0; return kCandBadM;  // optimizer.hpp:65-66 invalid_argument
  }
}

}  // namespace miso_b200

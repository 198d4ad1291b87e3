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

template <int M, bool kAll>
__device__ __forceinline__ int search_fixed(const double (&v)[M][5], double& best, uint64_t en0,
                                            uint64_t en1, bool tree) {
#define MISO_B200_SEARCH_CASE(MM)                                                  \
  if constexpr (M == MM)                                                            \
    return tree ? search_m##MM##_tree<kAll>(reinterpret_cast<const double(&)[MM][5]>(v), best, en0, en1) \
                : search_m##MM##_seq<kAll>(reinterpret_cast<const double(&)[MM][5]>(v), best, en0, en1);
  MISO_B200_SEARCH_CASE(1)
  MISO_B200_SEARCH_CASE(2)
  MISO_B200_SEARCH_CASE(3)
  MISO_B200_SEARCH_CASE(4)
  MISO_B200_SEARCH_CASE(5)
  MISO_B200_SEARCH_CASE(6)
  MISO_B200_SEARCH_CASE(7)
#undef MISO_B200_SEARCH_CASE
  return -1;
}

// Scores one instance whose m x 5 speed rows start at `row` (any address space). Only the
// slice kinds some size-M candidate uses are loaded (kKindsUsed). The tournament variant is
// used unless a loaded speed exceeds 2^1020: below that no sum of <= 7 speeds can reach +inf,
// so no inf + (-inf poison) = NaN can appear; otherwise the rank-ordered scan (where a NaN
// never wins) is the exact rule. Returns the candidate id or kCandInfeasible; *obj = objective.
template <int M, bool kAll, class Ptr>
__device__ __forceinline__ uint8_t search_rows(Ptr row, uint64_t en0, uint64_t en1, double* obj) {
  constexpr uint32_t kUsed = kKindsUsed[M];
  const double big = 0x1p1020;
  double v[M][5];
  bool has_inf = false;
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (kUsed & (1u << k)) {
        const double x = row[i * 5 + k];
        has_inf |= (x > big);
        v[i][k] = poison(x);
      } else {
        v[i][k] = 0.0;  // never referenced by a size-M candidate
      }
    }
  double best = __longlong_as_double(0xFFF0000000000000ll);
  int c = search_fixed<M, kAll>(v, best, en0, en1, !has_inf);
  *obj = c < 0 ? 0.0 : best;
  return c < 0 ? kCandInfeasible : static_cast<uint8_t>(c);
}

template <bool kAll, class Ptr>
__device__ __forceinline__ uint8_t search_any(Ptr row, int m, uint64_t en0, uint64_t en1,
                                              double* obj) {
  switch (m) {
    case 1: return search_rows<1, kAll>(row, en0, en1, obj);
    case 2: return search_rows<2, kAll>(row, en0, en1, obj);
    case 3: return search_rows<3, kAll>(row, en0, en1, obj);
    case 4: return search_rows<4, kAll>(row, en0, en1, obj);
    case 5: return search_rows<5, kAll>(row, en0, en1, obj);
    case 6: return search_rows<6, kAll>(row, en0, en1, obj);
    case 7: return search_rows<7, kAll>(row, en0, en1, obj);
    default: *obj = 0.0; return kCandBadM;  // optimizer.hpp:65-66 invalid_argument
  }
}

}  // namespace miso_b200

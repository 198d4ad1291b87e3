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

// optimize_partition for one roster, warp-parallel (rows: m x 5 in shared memory; all 32 lanes
// call it). Lane l scores candidates kCandBase[m] + l (+ 32): the job-order DADD sum of search_rows with
// invalid speeds poisoned to -inf; the winner is the largest objective, ties to the lowest
// candidate id (= OptKey rank, optimizer.hpp:46-51), and NaN / -inf sums never win -- the
// rank-ordered scan's rule, so the result is the same bits as search_any.
template <int M>
__device__ __forceinline__ void warp_score(const double* rows, const uint8_t (*place)[7], int c0,
                                           int c1, uint64_t en0, uint64_t en1, double& best,
                                           int& bc) {
  for (int c = c0 + static_cast<int>(threadIdx.x & 31); c < c1; c += 32) {
    const bool en = c < 64 ? ((en0 >> c) & 1ull) : ((en1 >> (c - 64)) & 1ull);
    uint8_t p[M];
#pragma unroll
    for (int i = 0; i < M; ++i) p[i] = place[c][i];
    double sum = poison(rows[p[0]]);
#pragma unroll
    for (int i = 1; i < M; ++i) sum = sum + poison(rows[i * 5 + p[i]]);
    if (en && sum > best) {  // ids rise within a lane: strict '>' keeps the lowest
      best = sum;
      bc = c;
    }
  }
}

__device__ __forceinline__ uint8_t warp_search(const double* rows, int m, uint64_t en0,
                                               uint64_t en1, const uint8_t (*place)[7],
                                               double* obj) {
  if (m < 1 || m > 7) {
    *obj = 0.0;
    return kCandBadM;  // optimizer.hpp:65-66 invalid_argument
  }
  double best = __longlong_as_double(0xFFF0000000000000ll);
  int bc = kCandInfeasible;
  // kCandBase[m], kCandBase[m + 1] packed one byte per m
  constexpr uint64_t kBase = uint64_t(kCandBase[1]) | uint64_t(kCandBase[2]) << 8 |
                             uint64_t(kCandBase[3]) << 16 | uint64_t(kCandBase[4]) << 24 |
                             uint64_t(kCandBase[5]) << 32 | uint64_t(kCandBase[6]) << 40 |
                             uint64_t(kCandBase[7]) << 48 | uint64_t(kCandBase[8]) << 56;
  const int c0 = static_cast<int>((kBase >> (8 * (m - 1))) & 0xff);
  const int c1 = static_cast<int>((kBase >> (8 * m)) & 0xff);
  switch (m) {
    case 1: warp_score<1>(rows, place, c0, c1, en0, en1, best, bc); break;
    case 2: warp_score<2>(rows, place, c0, c1, en0, en1, best, bc); break;
    case 3: warp_score<3>(rows, place, c0, c1, en0, en1, best, bc); break;
    case 4: warp_score<4>(rows, place, c0, c1, en0, en1, best, bc); break;
    case 5: warp_score<5>(rows, place, c0, c1, en0, en1, best, bc); break;
    case 6: warp_score<6>(rows, place, c0, c1, en0, en1, best, bc); break;
    default: warp_score<7>(rows, place, c0, c1, en0, en1, best, bc); break;
  }
  // Warp argmax on the objective's bits: a valid objective is positive (+inf included), where
  // the IEEE order is the unsigned order of the bit patterns and equality is bit equality;
  // no valid candidate = key 0. Then the lowest id among the lanes holding the maximum.
  const uint64_t key = bc == kCandInfeasible ? 0ull : static_cast<uint64_t>(__double_as_longlong(best));
  const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const unsigned id = __reduce_min_sync(0xffffffffu, hi == mhi && lo == mlo ? unsigned(bc) : 0xffu);
  if ((mhi | mlo) == 0u) {
    *obj = 0.0;
    return kCandInfeasible;
  }
  *obj = __longlong_as_double(static_cast<long long>((uint64_t(mhi) << 32) | mlo));
  return static_cast<uint8_t>(id);
}

}  // namespace miso_b200

// search_kernel.cu -- batched partition search (kernel (b)), one thread per instance.
//
// Data flow per CTA tile of kTile consecutive instances:
//   1. offsets[t0 .. t0+kTile] -> shared; m_i = offsets[i+1] - offsets[i].
//   2. the tile's packed speed rows (a contiguous byte range of the CSR speeds array) are
//      streamed into shared memory with coalesced 16-byte loads;
//   3. instances are bucketed by m inside the CTA (shared-memory counting sort) so the 32
//      threads of a warp run the same straight-line search_m<M> (no 7-way divergence);
//   4. each thread scores all candidates of its instance from registers (search.cuh);
//   5. decisions/objectives are staged in shared memory and written back coalesced.
// HBM traffic per instance = 40m (speeds) + 4 (offset) + 1 (cand) + 8 (objective) bytes.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "search.cuh"

namespace miso_b200 {

constexpr int kTile = 256;
constexpr int kMaxRowsPerTile = kTile * 7;
constexpr size_t kStageBytes = size_t(kMaxRowsPerTile) * 5 * sizeof(double) + 16;

__global__ void __launch_bounds__(kTile) optimize_tile_kernel(
    const double* __restrict__ speeds, const uint32_t* __restrict__ offsets, uint64_t n,
    uint8_t* __restrict__ cand_out, double* __restrict__ obj_out, uint64_t en0, uint64_t en1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_off[kTile + 1];
  __shared__ int s_cnt[8];
  __shared__ int s_base[8];
  __shared__ uint16_t s_order[kTile];
  __shared__ double s_obj[kTile];
  __shared__ uint8_t s_cand[kTile];

  const int tid = threadIdx.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * kTile;
  const int cnt = static_cast<int>(n - t0 < uint64_t(kTile) ? n - t0 : uint64_t(kTile));

  if (tid <= cnt) s_off[tid] = __ldg(offsets + t0 + tid);
  if (tid == 0 && cnt == kTile) s_off[kTile] = __ldg(offsets + t0 + kTile);
  if (tid < 8) s_cnt[tid] = 0;
  __syncthreads();

  const uint32_t j0 = s_off[0];
  const uint32_t njobs = s_off[cnt] - j0;
  const bool staged = njobs <= uint32_t(kMaxRowsPerTile) && s_off[cnt] >= j0;

  // --- 2. stage the tile's speed rows: 16-byte chunks, aligned on the absolute address ---
  const double* gsrc = speeds + size_t(j0) * 5;
  const unsigned char* gbytes = reinterpret_cast<const unsigned char*>(gsrc);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(gbytes);
  const uintptr_t abase = a0 & ~uintptr_t(15);
  const int lead = static_cast<int>(a0 - abase);  // 0 or 8 (rows are 8-byte aligned)
  double* srows = reinterpret_cast<double*>(smem_raw + lead);
  if (staged) {
    const size_t nbytes = size_t(njobs) * 40;
    const size_t nchunks = (lead + nbytes + 15) / 16;
    const uint4* g4 = reinterpret_cast<const uint4*>(abase);
    uint4* s4 = reinterpret_cast<uint4*>(smem_raw);
    // First and last chunk may straddle the array ends: copy those bytes as doubles.
    for (size_t c = tid; c < nchunks; c += kTile) {
      if ((c == 0 && lead != 0) || (c == nchunks - 1 && ((lead + nbytes) & 15) != 0)) continue;
      s4[c] = __ldg(g4 + c);
    }
    if (tid == 0 && lead != 0 && njobs > 0) srows[0] = __ldg(gsrc);
    if (tid == 1 && ((lead + nbytes) & 15) != 0 && njobs > 0)
      srows[size_t(njobs) * 5 - 1] = __ldg(gsrc + size_t(njobs) * 5 - 1);
  }

  // --- 3. bucket instances by m ---
  int my_m = 0, my_rank = 0;
  if (tid < cnt) {
    uint32_t mm = s_off[tid + 1] - s_off[tid];
    my_m = (mm >= 1 && mm <= 7) ? static_cast<int>(mm) : 0;
    my_rank = atomicAdd(&s_cnt[my_m], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int b = 0;
    for (int k = 0; k < 8; ++k) { s_base[k] = b; b += s_cnt[k]; }
  }
  __syncthreads();
  if (tid < cnt) s_order[s_base[my_m] + my_rank] = static_cast<uint16_t>(tid);
  __syncthreads();

  // --- 4. search ---
  if (tid < cnt) {
    const int l = s_order[tid];
    const uint32_t o = s_off[l];
    const uint32_t mm = s_off[l + 1] - o;
    const int m = (mm >= 1 && mm <= 7) ? static_cast<int>(mm) : 0;
    double obj = 0.0;
    uint8_t c;
    // Rows outside the staged range only occur with non-monotonic (malformed) offsets.
    if (staged && o >= j0 && o - j0 + uint32_t(m) <= njobs)
      c = search_any(srows + size_t(o - j0) * 5, m, en0, en1, &obj);
    else
      c = search_any(speeds + size_t(o) * 5, m, en0, en1, &obj);
    s_cand[l] = c;
    s_obj[l] = obj;
  }
  __syncthreads();

  // --- 5. coalesced write-back ---
  if (tid < cnt) {
    cand_out[t0 + tid] = s_cand[tid];
    obj_out[t0 + tid] = s_obj[tid];
  }
}

cudaError_t launch_optimize(const double* speeds, const uint32_t* offsets, uint64_t n,
                            uint8_t* cand, double* obj, uint64_t en0, uint64_t en1,
                            cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(optimize_tile_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kStageBytes));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const uint64_t blocks = (n + kTile - 1) / kTile;
  optimize_tile_kernel<<<static_cast<unsigned>(blocks), kTile, kStageBytes, stream>>>(
      speeds, offsets, n, cand, obj, en0, en1);
  return cudaGetLastError();
}

}  // namespace miso_b200

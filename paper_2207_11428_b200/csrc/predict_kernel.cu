// predict_kernel.cu -- kernel (a): batched MPS->MIG predictor, and the fused
// predictor -> effective_speed -> partition search kernel (the per-GPU decision of
// finish_profiling + reopt_and_apply, sim.hpp:691-733, for many rosters at once).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "predict.cuh"
#include "search.cuh"

namespace miso_b200 {

// ---------------------------------------------------------------------------------------
// Batched predictor: one thread per profile column. Column j belongs to group j / cpg as its
// column j % cpg; the group's call nonce is first_nonce + j / cpg (pad_to_seven places real
// jobs in columns 0..cpg-1, profiles.hpp:106-113). In: truth (f7,f4,f3) per column. Out: the
// five estimated speeds per column in kind order 1g..7g. Rows are staged through shared
// memory so global loads and stores are coalesced.
// ---------------------------------------------------------------------------------------
constexpr int kPredBlock = 256;

__global__ void __launch_bounds__(kPredBlock) predict_batch_kernel(
    const double* __restrict__ truth3, uint64_t ncols, int cpg, uint64_t first_nonce,
    uint64_t rng_seed, int noisy, double target_mae, ModelW w, double* __restrict__ out5) {
  __shared__ double s_in[kPredBlock * 3];
  __shared__ double s_out[kPredBlock * 5];
  const uint64_t j0 = uint64_t(blockIdx.x) * kPredBlock;
  const int cnt = static_cast<int>(ncols - j0 < uint64_t(kPredBlock) ? ncols - j0 : uint64_t(kPredBlock));
  for (int i = threadIdx.x; i < cnt * 3; i += kPredBlock) s_in[i] = truth3[j0 * 3 + i];
  __syncthreads();
  if (static_cast<int>(threadIdx.x) < cnt) {
    const uint64_t j = j0 + threadIdx.x;
    const uint64_t g = j / static_cast<uint64_t>(cpg);
    const int c = static_cast<int>(j - g * static_cast<uint64_t>(cpg));
    const double* t = s_in + threadIdx.x * 3;
    predict_column(t[0], t[1], t[2], c, rng_seed, first_nonce + g, noisy != 0, target_mae, w,
                   s_out + threadIdx.x * 5);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt * 5; i += kPredBlock) out5[j0 * 5 + i] = s_out[i];
}

cudaError_t launch_predict(const double* truth3, uint64_t ncols, int cpg, uint64_t first_nonce,
                           uint64_t rng_seed, int noisy, double target_mae, const double* w2,
                           const double* w1, double* out5, cudaStream_t stream) {
  if (ncols == 0) return cudaSuccess;
  ModelW w;
  for (int i = 0; i < 4; ++i) {
    w.w2[i] = w2[i];
    w.w1[i] = w1[i];
  }
  const uint64_t blocks = (ncols + kPredBlock - 1) / kPredBlock;
  predict_batch_kernel<<<static_cast<unsigned>(blocks), kPredBlock, 0, stream>>>(
      truth3, ncols, cpg, first_nonce, rng_seed, noisy, target_mae, w, out5);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Fused decision kernel: per instance (a roster of m <= 7 jobs in columns 0..m-1), predict
// every job's speeds (call nonce = nonce[i]), zero them by memory demand / QoS floor
// (effective_speed) and run the partition search -- entirely on chip, one CTA tile of
// kDecTile instances: phase 1 one thread per job (predictor, the expensive part), phase 2
// one thread per instance over the m-bucketed tile (search.cuh).
// Per job in: truth (f7,f4,f3), mem_gb (u8), qos kind (int8, -1 = none).
// ---------------------------------------------------------------------------------------
constexpr int kDecTile = 128;

template <bool kAll>
__global__ void __launch_bounds__(kDecTile) decide_tile_kernel(
    const double* __restrict__ truth3, const uint8_t* __restrict__ mem_gb,
    const int8_t* __restrict__ qos_kind, const uint32_t* __restrict__ offsets,
    const uint64_t* __restrict__ nonce, uint64_t n, uint64_t rng_seed, int noisy,
    double target_mae, ModelW w, uint64_t en0, uint64_t en1, uint8_t* __restrict__ cand_out,
    double* __restrict__ obj_out, double* __restrict__ est_out) {
  __shared__ uint32_t s_off[kDecTile + 1];
  __shared__ double s_rows[kDecTile * 7 * 5];
  __shared__ int s_cnt[8], s_base[8];
  __shared__ uint16_t s_order[kDecTile];
  const int tid = threadIdx.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * kDecTile;
  const int cnt = static_cast<int>(n - t0 < uint64_t(kDecTile) ? n - t0 : uint64_t(kDecTile));
  if (tid <= cnt) s_off[tid] = offsets[t0 + tid];
  if (tid == 0 && cnt == kDecTile) s_off[kDecTile] = offsets[t0 + kDecTile];
  if (tid < 8) s_cnt[tid] = 0;
  __syncthreads();
  const uint32_t j0 = s_off[0];
  const uint32_t njobs = s_off[cnt] - j0;
  const bool tile_ok = s_off[cnt] >= j0 && njobs <= uint32_t(kDecTile * 7);

  // phase 1: one thread per job (jobs of malformed tiles are handled in phase 2 directly)
  if (tile_ok) {
    for (uint32_t jj = tid; jj < njobs; jj += kDecTile) {
      int lo = 0, hi = cnt;  // instance owning job j0+jj: last l with s_off[l] <= j0+jj
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= j0 + jj) lo = mid; else hi = mid;
      }
      const int col = static_cast<int>(j0 + jj - s_off[lo]);
      const uint64_t j = uint64_t(j0) + jj;
      double e[5];
      predict_column(truth3[3 * j], truth3[3 * j + 1], truth3[3 * j + 2], col, rng_seed,
                     nonce[t0 + lo], noisy != 0, target_mae, w, e);
      const int mem = mem_gb[j], qk = qos_kind[j];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const double v = effective_speed(e[k], k, mem, qk);
        s_rows[jj * 5 + k] = v;
        if (est_out) est_out[j * 5 + k] = v;
      }
    }
  }

  // phase 2: bucket by m, one thread per instance
  int my_m = 0, my_rank = 0;
  if (tid < cnt) {
    const uint32_t mm = s_off[tid + 1] - s_off[tid];
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
  if (tid < cnt) {
    const int l = s_order[tid];
    const uint32_t o = s_off[l];
    const uint32_t mm = s_off[l + 1] - o;
    const int m = (mm >= 1 && mm <= 7) ? static_cast<int>(mm) : 0;
    double ob = 0.0;
    uint8_t c = kCandBadM;
    if (tile_ok && m > 0) {
      c = search_any<kAll>(s_rows + size_t(o - j0) * 5, m, en0, en1, &ob);
    } else if (m > 0) {  // malformed tile (non-monotone offsets): predict this roster here
      double rows[7 * 5];
      for (int jj = 0; jj < m; ++jj) {
        const uint64_t j = uint64_t(o) + jj;
        double e[5];
        predict_column(truth3[3 * j], truth3[3 * j + 1], truth3[3 * j + 2], jj, rng_seed,
                       nonce[t0 + l], noisy != 0, target_mae, w, e);
        for (int k = 0; k < 5; ++k) {
          rows[jj * 5 + k] = effective_speed(e[k], k, mem_gb[j], qos_kind[j]);
          if (est_out) est_out[j * 5 + k] = rows[jj * 5 + k];
        }
      }
      c = search_any<kAll>(rows, m, en0, en1, &ob);
    }
    cand_out[t0 + l] = c;
    obj_out[t0 + l] = ob;
  }
}

cudaError_t launch_decide(const double* truth3, const uint8_t* mem_gb, const int8_t* qos_kind,
                          const uint32_t* offsets, const uint64_t* nonce, uint64_t n,
                          uint64_t rng_seed, int noisy, double target_mae, const double* w2,
                          const double* w1, uint64_t en0, uint64_t en1, uint8_t* cand,
                          double* obj, double* est_out, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  ModelW w;
  for (int i = 0; i < 4; ++i) {
    w.w2[i] = w2[i];
    w.w1[i] = w1[i];
  }
  const bool all = en0 == ~0ull && en1 == (1ull << (kNumCands - 64)) - 1;
  const uint64_t blocks = (n + kDecTile - 1) / kDecTile;
  if (all)
    decide_tile_kernel<true><<<static_cast<unsigned>(blocks), kDecTile, 0, stream>>>(
        truth3, mem_gb, qos_kind, offsets, nonce, n, rng_seed, noisy, target_mae, w, en0, en1,
        cand, obj, est_out);
  else
    decide_tile_kernel<false><<<static_cast<unsigned>(blocks), kDecTile, 0, stream>>>(
        truth3, mem_gb, qos_kind, offsets, nonce, n, rng_seed, noisy, target_mae, w, en0, en1,
        cand, obj, est_out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Single-roster latency path (config 1, miso_b200_decide): the whole roster travels as kernel
// parameters (no device-side reads of host or global input), one warp predicts -- lane
// 2c + e perturbs entry e (4g, 3g) of column c, so the two mt19937_64 seeding chains of a
// column run side by side -- lane 0 searches, and the results plus a completion sequence
// number are stored straight into mapped pinned host memory (the host spins on `seq`).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(32) decide_one_kernel(DecideOneArgs a, DecideOneOut* out) {
  __shared__ double s_rows[7 * 5];
  __shared__ double s_pert[7][2];
  const int lane = threadIdx.x;
  const int m = a.m;
  // perturbed 4g / 3g entries (profiles.hpp:234-244), one per lane
  if (lane < 2 * m) {
    const int c = lane >> 1, e = lane & 1;
    const double truth = a.truth[c][1 + e];
    double v = truth;
    if (a.noisy) {
      const uint64_t base = mix_seed(a.rng_seed, a.nonce);
      v = perturb_speed(truth, a.target_mae, mix_seed(base, static_cast<uint64_t>(c) * 8 + 1 + e));
    }
    s_pert[c][e] = v;
  }
  __syncwarp();
  if (lane < m) {
    // re-anchor, clamp and extrapolate exactly as predict_column (oracle-mode inputs)
    ModelW w;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w.w2[i] = a.w2[i];
      w.w1[i] = a.w1[i];
    }
    double e5[5];
    predict_column(a.truth[lane][0], s_pert[lane][0], s_pert[lane][1], lane, 0, 0, false, 0.0,
                   w, e5);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double v = effective_speed(e5[k], k, a.mem[lane], a.qos[lane]);
      s_rows[lane * 5 + k] = v;
      out->est[lane * 5 + k] = v;
    }
  }
  __syncwarp();
  if (lane == 0) {
    double ob = 0.0;
    const bool all = a.en0 == ~0ull && a.en1 == (1ull << (kNumCands - 64)) - 1;
    const uint8_t c = all ? search_any<true>(s_rows, m, a.en0, a.en1, &ob)
                          : search_any<false>(s_rows, m, a.en0, a.en1, &ob);
    out->cand = c;
    out->obj = ob;
  }
  __threadfence_system();
  __syncwarp();
  if (lane == 0) *reinterpret_cast<volatile uint64_t*>(&out->seq) = a.seq;
}

cudaError_t launch_decide_one(const DecideOneArgs& a, DecideOneOut* out, cudaStream_t stream) {
  decide_one_kernel<<<1, 32, 0, stream>>>(a, out);
  return cudaGetLastError();
}

}  // namespace miso_b200

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
    predict_column(t[0], t[1], t[2], c, rng_seed, first_nonce + g, noisy == 1, target_mae, w,
                   s_out + threadIdx.x * 5, noisy != 2);
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
// Single-roster latency path (config 1, miso_b200_decide). One warp predicts -- lane 2c + e
// perturbs entry e (4g, 3g) of column c -- lane 0 searches, and the result record (est rows,
// objective, candidate, request number, check word) is stored straight into mapped pinned
// host memory by consecutive lanes; the host accepts it when the check word matches.
// decide_one_kernel takes the roster as a kernel parameter (one launch per call);
// decide_server_kernel stays resident and polls a mailbox (capi.cu, miso_b200_decide).
// ---------------------------------------------------------------------------------------
// The noise draws of one predictor call: entry e (4g, 3g) of column c < 7 is lane 2c + e.
// Only the call's (rng_seed, nonce) picks them (profiles.hpp:234-244), so the server's second
// warp computes them ahead for the next nonce (decide_server_kernel).
__device__ __forceinline__ NoiseDraw call_draw(uint64_t rng_seed, uint64_t nonce, int lane) {
  const int c = lane >> 1, e = lane & 1;
  const uint64_t base = mix_seed(rng_seed, nonce);
  uint64_t r[3];
  mt64_first3(mix_seed(base, static_cast<uint64_t>(c) * 8 + 1 + e), r);
  return noise_draw(r);
}

// pre: this lane's draw when the caller has it (the server's draw-ahead), else nullptr.
// place: the candidate placement table (shared-memory copy in the server).
__device__ __forceinline__ void decide_one_body(const DecideOneArgs& a, DecideOneOut& o,
                                                const uint8_t (*place)[7],
                                                uint64_t* cyc = nullptr,
                                                const NoiseDraw* pre = nullptr) {
  __shared__ double s_pert[7][2];
  const int lane = threadIdx.x;
  const int m = a.m;
  if (a.noisy == kSearchOnly) {  // optimize_partition alone: the speeds come packed in the args
    const double* sp = &a.truth[0][0];
    const int stride = m == 1 ? 5 : 4;  // 7g is used by the m = 1 entry "7g" only
    if (lane < 7) {
#pragma unroll
      for (int k = 0; k < 5; ++k)
        o.est[lane * 5 + k] = lane < m && (k < 4 || m == 1) ? sp[lane * stride + k] : 0.0;
    }
    __syncwarp();
    double ob;
    const uint8_t c = warp_search(o.est, m, a.en0, a.en1, place, &ob);
    if (lane == 0) {
      o.cand = c;
      o.obj = ob;
      o.seq = a.seq;
    }
    __syncwarp();
    return;
  }
  const long long c0 = clock64();
  // perturbed 4g / 3g entries (profiles.hpp:234-244), one per lane
  if (lane < 2 * m) {
    const int c = lane >> 1, e = lane & 1;
    const double truth = a.truth[c][1 + e];
    double v = truth;
    if (a.noisy && a.target_mae > 0.0) {  // (target_mae <= 0: perturb_speed returns the truth)
      v = perturb_apply(truth, a.target_mae, pre ? *pre : call_draw(a.rng_seed, a.nonce, lane));
    }
    s_pert[c][e] = v;
  }
  __syncwarp();
  const long long c1 = clock64();
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
    for (int k = 0; k < 5; ++k) o.est[lane * 5 + k] = effective_speed(e5[k], k, a.mem[lane], a.qos[lane]);
  } else if (lane < 7) {
#pragma unroll
    for (int k = 0; k < 5; ++k) o.est[lane * 5 + k] = 0.0;
  }
  __syncwarp();
  const long long c2 = clock64();
  double ob;
  const uint8_t c = warp_search(o.est, m, a.en0, a.en1, place, &ob);
  if (lane == 0) {
    o.cand = c;
    o.obj = ob;
    o.seq = a.seq;
  }
  __syncwarp();
  if (cyc && lane == 0) {  // timing probe: perturb, predict, search cycles
    cyc[0] = uint64_t(c1 - c0);
    cyc[1] = uint64_t(c2 - c1);
    cyc[2] = uint64_t(clock64() - c2);
  }
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Store the shared record o to out (mapped host memory) with its check word; no fence: the
// host re-reads until the check matches.
__device__ __forceinline__ void decide_publish(const DecideOneOut& o, DecideOneOut* out, int m) {
  const int lane = threadIdx.x;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(&o);
  const int n = kOutEst + 5 * m;  // the record's live words: header + m est rows
  const uint64_t mine = lane < n ? w[lane] : 0;
  uint64_t part = lane < n && lane != kOutCheck ? mbx_mix(mine, uint64_t(lane)) : 0;
  const uint64_t extra = lane + 32 < n ? w[lane + 32] : 0;
  if (lane + 32 < n) part += mbx_mix(extra, uint64_t(lane + 32));
  const uint64_t check = warp_sum_u64(part);
  volatile uint64_t* dst = reinterpret_cast<volatile uint64_t*>(out);
  if (lane < n) dst[lane] = lane == kOutCheck ? check : mine;
  if (lane + 32 < n) dst[lane + 32] = extra;
}

__global__ void __launch_bounds__(32) decide_one_kernel(DecideOneArgs a, DecideOneOut* out) {
  __shared__ DecideOneOut s_o;
  decide_one_body(a, s_o, kCandPlaceD);
  decide_publish(s_o, out, a.noisy == kSearchOnly ? 0 : a.m);  // search-only: header alone
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Resident form: warp 0 polls the mailbox (mapped pinned host memory). Every poll is one
// PCIe round trip that fetches the whole mailbox (lanes 0..19, 16 B each); a request is
// taken when args.seq differs from the last one served and the check word matches the
// fetched words (a fetch that raced the host's writes fails the check and is repeated). The
// server exits when the host sets `stop`, after idle_ns without a request, or after life_ns
// in total; the host relaunches it on demand.
//
// Warp 1 computes ahead: after each request warp 0 posts (rng_seed, nonce + 1) -- callers
// number their predictor calls consecutively (SimEngine's call nonce) -- and warp 1 makes
// sure the draws of nonces +1 and +2 are in a 4-slot ring (lanes 0..13 and 14..27 run the
// two calls' 158-step seeding chains plus log/cos side by side, ~75% of a request's
// compute). A request finds its draws by nonce; each slot is a seqlock (odd version = being
// written), so a slot rewritten while warp 0 read it is detected and warp 0 computes the
// draws itself -- as it does for any call nobody computed ahead. Either way the draws are the
// same bits.
// Every shared word the two warps hand to each other is accessed with shared-memory atomics
// (relaxed, ordered by __threadfence_block): the protocol is flag/seqlock based rather than
// barrier based, and atomics make each cross-warp access well defined (and visible as such to
// compute-sanitizer's racecheck).
constexpr int kAheadSlots = 4, kAhead = 2;

struct DrawSlot {
  unsigned long long n01[14];            // double bits
  unsigned long long rng_seed, nonce;
  unsigned coins;                        // bit l = lane l's coin
  unsigned ver;                          // seqlock version; odd = being written (or never written)
};

struct DrawAhead {
  DrawSlot slot[kAheadSlots];
  unsigned long long want_seed, want_nonce;
  unsigned posted, quit;
};

__device__ __forceinline__ unsigned long long sh_ld(unsigned long long* p) { return atomicAdd(p, 0ull); }
__device__ __forceinline__ unsigned sh_ld(unsigned* p) { return atomicAdd(p, 0u); }
__device__ __forceinline__ void sh_st(unsigned long long* p, unsigned long long v) { atomicExch(p, v); }
__device__ __forceinline__ void sh_st(unsigned* p, unsigned v) { atomicExch(p, v); }

// Control words are read by lane 0 and broadcast: per-lane atomics are separate reads, and a
// warp must branch on one snapshot.
__device__ __forceinline__ unsigned long long bcast_ld(unsigned long long* p) {
  unsigned long long v = 0;
  if ((threadIdx.x & 31) == 0) v = sh_ld(p);
  return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ unsigned bcast_ld(unsigned* p) {
  unsigned v = 0;
  if ((threadIdx.x & 31) == 0) v = sh_ld(p);
  return __shfl_sync(0xffffffffu, v, 0);
}

__device__ __forceinline__ void draw_ahead_worker(DrawAhead& da) {
  const int lane = threadIdx.x & 31;
  unsigned served = 0;
  for (;;) {
    unsigned posted;
    for (;;) {
      if (bcast_ld(&da.quit)) return;
      posted = bcast_ld(&da.posted);
      if (posted != served) break;
      __nanosleep(128);
    }
    served = posted;
    __threadfence_block();
    // (a post racing these reads only mixes keys; the slot records the key it computed for)
    const uint64_t rs = bcast_ld(&da.want_seed), first = bcast_ld(&da.want_nonce);
    const int k = lane / 14, l = lane % 14;
    bool need[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      DrawSlot& sl = da.slot[(first + q) % kAheadSlots];
      need[q] = (bcast_ld(&sl.ver) & 1u) || bcast_ld(&sl.nonce) != first + q ||
                bcast_ld(&sl.rng_seed) != rs;
    }
    if (!need[0] && !need[1]) continue;
    NoiseDraw d{0.0, false};
    if (k < kAhead && need[k]) d = call_draw(rs, first + k, l);
    const uint32_t coins = __ballot_sync(0xffffffffu, d.coin);
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      if (!need[q]) continue;
      DrawSlot& sl = da.slot[(first + q) % kAheadSlots];
      if (lane == 0) {
        atomicOr(&sl.ver, 1u);
        __threadfence_block();
      }
      __syncwarp();
      if (k == q) sh_st(&sl.n01[l], static_cast<unsigned long long>(__double_as_longlong(d.n01)));
      if (lane == 0) {
        sh_st(&sl.coins, (coins >> (14 * q)) & 0x3fffu);
        sh_st(&sl.rng_seed, rs);
        sh_st(&sl.nonce, first + q);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&sl.ver, 1u);
      }
      __syncwarp();
    }
  }
}

// Warp 0: this lane's draw of call (rng_seed, nonce) from the ring, if a consistent copy is
// there (seqlock read by lane 0 around the lanes' data reads; warp-uniform result).
__device__ __forceinline__ bool take_ahead(DrawAhead& da, uint64_t rng_seed, uint64_t nonce,
                                           NoiseDraw& d) {
  const int lane = threadIdx.x & 31;
  DrawSlot& sl = da.slot[nonce % kAheadSlots];
  const unsigned v1 = bcast_ld(&sl.ver);
  __threadfence_block();
  if ((v1 & 1u) || bcast_ld(&sl.nonce) != nonce || bcast_ld(&sl.rng_seed) != rng_seed) return false;
  if (lane < 14) {
    d.n01 = __longlong_as_double(static_cast<long long>(sh_ld(&sl.n01[lane])));
    d.coin = (sh_ld(&sl.coins) >> lane) & 1u;
  }
  __syncwarp();
  __threadfence_block();
  return bcast_ld(&sl.ver) == v1;
}

__global__ void __launch_bounds__(64) decide_server_kernel(const DecideMailbox* mb,
                                                           DecideOneOut* out, uint64_t last,
                                                           uint64_t idle_ns, uint64_t life_ns,
                                                           uint64_t* stamps, uint32_t poll_ns) {
  __shared__ DecideOneArgs s_a;
  __shared__ DecideOneOut s_o;
  __shared__ DrawAhead da;
  __shared__ uint8_t s_place[kNumCands][7];
  for (int i = threadIdx.x; i < kNumCands * 7; i += blockDim.x)
    (&s_place[0][0])[i] = (&kCandPlaceD[0][0])[i];
  if (threadIdx.x < kAheadSlots) da.slot[threadIdx.x].ver = 1u;
  if (threadIdx.x == 0) {
    da.posted = 0;
    da.quit = 0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) {
    draw_ahead_worker(da);
    return;
  }
  const int lane = threadIdx.x;
  const uint64_t t0 = global_ns();
  uint64_t t_last = t0;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(mb);
  // The expected next call (rng_seed, nonce + 1) and, once the ring has it, its draws in
  // registers: fetched while a poll is in flight, so a matching request skips the ring read.
  bool want_pre = false, have_pre = false;
  uint64_t pre_seed = 0, pre_nonce = 0;
  NoiseDraw pre{0.0, false};
  auto poll = [&](unsigned long long& w0, unsigned long long& w1) {
    if (lane < 20)
      asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                   : "=l"(w0), "=l"(w1) : "l"(src + 2 * lane) : "memory");
  };
  // One fetched mailbox image: serve it if it holds a new request; true = exit.
  auto serve = [&](unsigned long long w0, unsigned long long w1) -> bool {
    if (want_pre && !have_pre) have_pre = take_ahead(da, pre_seed, pre_nonce, pre);
    const uint64_t seq = __shfl_sync(0xffffffffu, (kArgSeqWord & 1) ? w1 : w0, kArgSeqWord >> 1);
    const uint64_t stop = __shfl_sync(0xffffffffu, w1, 19);
    if (stop) return true;
    if (seq != last) {
      const uint64_t ts0 = stamps ? global_ns() : 0;
      uint64_t part = 0;
      if (2 * lane < kArgWords) part += mbx_mix(w0, uint64_t(2 * lane));
      if (2 * lane + 1 < kArgWords) part += mbx_mix(w1, uint64_t(2 * lane + 1));
      const uint64_t check = __shfl_sync(0xffffffffu, w0, kArgWords >> 1);  // word kArgWords
      if (warp_sum_u64(part) != check) return false;  // torn fetch: poll again
      uint64_t* dst = reinterpret_cast<uint64_t*>(&s_a);
      if (2 * lane < kArgWords) dst[2 * lane] = w0;
      if (2 * lane + 1 < kArgWords) dst[2 * lane + 1] = w1;
      __syncwarp();
      const uint64_t ts1 = stamps ? global_ns() : 0;
      const long long c1 = clock64();
      if (s_a.noisy == kSearchOnly) {  // optimize_partition request: no predictor, no draw-ahead
        decide_one_body(s_a, s_o, s_place);
        decide_publish(s_o, out, 0);
        last = seq;
        __syncwarp();
        t_last = global_ns();
        return false;
      }
      NoiseDraw mine = pre;
      bool hit = false;
      if (s_a.noisy) {
        hit = have_pre && s_a.rng_seed == pre_seed && s_a.nonce == pre_nonce;
        if (!hit) hit = take_ahead(da, s_a.rng_seed, s_a.nonce, mine);
      }
      decide_one_body(s_a, s_o, s_place, stamps ? stamps + 8 : nullptr, hit ? &mine : nullptr);
      want_pre = true;
      have_pre = false;
      pre_seed = s_a.rng_seed;
      pre_nonce = s_a.nonce + 1;
      const uint64_t ts2 = stamps ? global_ns() : 0;
      const long long c2 = clock64();
      decide_publish(s_o, out, s_a.m);
      // post the next calls' draws (warp 1 picks the new generation up when it is idle)
      if (lane == 0) {
        sh_st(&da.want_seed, s_a.rng_seed);
        sh_st(&da.want_nonce, s_a.nonce + 1);
        __threadfence_block();
        atomicAdd(&da.posted, 1u);
      }
      if (stamps && lane == 0) {  // timing probe (tools/decide_probe.cu)
        stamps[0] = ts0;
        stamps[1] = ts1;
        stamps[2] = ts2;
        stamps[3] = global_ns();
        stamps[4] = hit;
        stamps[5] = uint64_t(c2 - c1);
        stamps[6] = uint64_t(clock64() - c2);
      }
      last = seq;
      __syncwarp();
      t_last = global_ns();
      return false;
    }
    const uint64_t now = global_ns();
    return now - t_last > idle_ns || now - t0 > life_ns;
  };
  // Two polls in flight, issued poll_ns apart: the mailbox is sampled twice per PCIe round
  // trip, so a request waits about a quarter round trip less to be noticed.
  unsigned long long a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  poll(a0, a1);
  for (;;) {
    if (poll_ns) __nanosleep(poll_ns);
    poll(b0, b1);
    if (serve(a0, a1)) break;
    if (poll_ns) __nanosleep(poll_ns);
    poll(a0, a1);
    if (serve(b0, b1)) break;
  }
  if (lane == 0) sh_st(&da.quit, 1u);
}

cudaError_t launch_decide_one(const DecideOneArgs& a, DecideOneOut* out, cudaStream_t stream) {
  decide_one_kernel<<<1, 32, 0, stream>>>(a, out);
  return cudaGetLastError();
}

cudaError_t launch_decide_server(const DecideMailbox* mb, DecideOneOut* out, uint64_t last,
                                 uint64_t idle_ns, uint64_t life_ns, cudaStream_t stream,
                                 uint64_t* stamps, uint32_t poll_ns) {
  decide_server_kernel<<<1, 64, 0, stream>>>(mb, out, last, idle_ns, life_ns, stamps, poll_ns);
  return cudaGetLastError();
}

}  // namespace miso_b200

// search_kernel.cu -- batched partition search (kernel (b)), one thread per instance.
//
// Default path: optimize_pipe_kernel, a persistent warp-specialized pipeline (see below): a
// producer warp streams kT-instance tiles (offsets + CSR speed rows) into a kS-stage
// shared-memory ring with TMA bulk copies; consumer groups bucket each tile by job count m and
// search one instance per thread from registers (search.cuh).
// Fallback (speeds not 16-byte aligned, or MISO_B200_SIMPLE_SEARCH=1): optimize_tile_kernel,
// one CTA per tile with a synchronous staged copy.
//
// HBM traffic per instance = 40m (speeds) + 4 (offset) + 1 (decision) + 8 (objective) bytes.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "search.cuh"
#include "tma.cuh"

#ifndef MISO_B200_TRACE
#define MISO_B200_TRACE 0
#endif

namespace miso_b200 {

#if MISO_B200_TRACE
// Debug timeline (tools/trace_search.cu): [blockIdx][event] = globaltimer.
__device__ unsigned long long g_trace[148][4096];
__device__ __forceinline__ void trace(int slot) {
  if (blockIdx.x < 148 && slot < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[blockIdx.x][slot] = t;
  }
}
#define TRACE(slot) trace(slot)
#else
#define TRACE(slot) ((void)0)
#endif

static bool force_simple_path() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MISO_B200_SIMPLE_SEARCH");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Programmatic dependent launch for the persistent search kernel (MISO_B200_NO_PDL=1 disables).
static bool use_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MISO_B200_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

__device__ __forceinline__ int valid_m(uint32_t mm) {
  return (mm >= 1 && mm <= 7) ? static_cast<int>(mm) : 0;
}

// ---------------------------------------------------------------------------------------
// Fallback: one-shot tile kernel.
// ---------------------------------------------------------------------------------------
constexpr int kTile = 256;
constexpr int kMaxRowsPerTile = kTile * 7;
constexpr size_t kTileStageBytes = size_t(kMaxRowsPerTile) * 5 * sizeof(double) + 16;

template <bool kAll>
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

  const double* gsrc = speeds + size_t(j0) * 5;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(gsrc);
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

  int my_m = 0, my_rank = 0;
  if (tid < cnt) {
    my_m = valid_m(s_off[tid + 1] - s_off[tid]);
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
    const int m = valid_m(s_off[l + 1] - o);
    double obj = 0.0;
    uint8_t c;
    // Rows outside the staged range only occur with non-monotonic (malformed) offsets.
    if (staged && o >= j0 && o - j0 + uint32_t(m) <= njobs)
      c = search_any<kAll>(srows + size_t(o - j0) * 5, m, en0, en1, &obj);
    else
      c = search_any<kAll>(speeds + size_t(o) * 5, m, en0, en1, &obj);
    s_cand[l] = c;
    s_obj[l] = obj;
  }
  __syncthreads();

  if (tid < cnt) {
    cand_out[t0 + tid] = s_cand[tid];
    obj_out[t0 + tid] = s_obj[tid];
  }
}

// ---------------------------------------------------------------------------------------
// Persistent warp-specialized TMA pipeline (default path).
//
//   producer warp: for each tile of kT instances, waits for a free stage of the kS-stage
//     shared-memory ring and issues two cp.async.bulk (TMA 1-D bulk) copies -- the tile's
//     kT+1 offsets and its contiguous speed rows -- completing on full[stage]. Tile boundaries
//     (offsets[t0], offsets[t0+cnt]) are prefetched 32 tiles at a time (lane l holds tile
//     k+l), so issuing never waits on a dependent global load.
//   kG consumer groups of kT threads take alternate tiles: bucket the tile by job count m
//     (shared-memory counting sort, so every warp runs one straight-line search_m<M>), search
//     one instance per thread from registers (search.cuh), release the stage (empty[stage]),
//     and flush the previous tile's decisions coalesced (double-buffered, 2 named barriers
//     per tile).
// ---------------------------------------------------------------------------------------
template <int kT, int kS, int kCap>
struct PipeLayout {
  static constexpr int kOffWords = ((kT + 1 + 3) / 4) * 4;
  static constexpr size_t kRowBytes = size_t(kCap) * 40 + 32;
  static constexpr size_t kStageBytes = ((kOffWords * 4 + kRowBytes + 127) / 128) * 128;
  static constexpr size_t kBytes = kStageBytes * kS + 128;
};

// The batches of one launch (kernel parameter space, read with dynamic indices through
// __grid_constant__): batch b owns global tiles tile0[b] .. tile0[b+1]-1 of kT instances each.
struct PipeBatches {
  const double* speeds[kMaxPipeBatches];
  const uint32_t* offsets[kMaxPipeBatches];
  uint8_t* cand[kMaxPipeBatches];
  double* obj[kMaxPipeBatches];
  uint64_t n[kMaxPipeBatches];
  uint64_t tile0[kMaxPipeBatches + 1];
  int nb;
};

#ifndef MISO_SEARCH_ALL_ARRIVE
#define MISO_SEARCH_ALL_ARRIVE 0
#endif
// Arrivals that release a stage: one per consumer warp (lane 0 after __syncwarp), or one per
// consumer thread with MISO_SEARCH_ALL_ARRIVE (the form compute-sanitizer racecheck can follow).
template <int kT>
constexpr uint32_t kEmptyArrivals = MISO_SEARCH_ALL_ARRIVE ? kT : kT / 32;

// Advances a batch cursor to the batch that owns global tile `tile` (tiles only grow per thread).
__device__ __forceinline__ int batch_of(const PipeBatches& B, uint64_t tile, int b) {
  while (B.tile0[b + 1] <= tile) ++b;
  return b;
}

// kPos: nibble m = position of job count m's bucket in the sorted tile (identity = ascending
// m). Warps straddle bucket boundaries and run both paths, so an order that puts cheap m next
// to expensive m shortens the slowest warp of a tile.
template <int kT, int kS, int kCap, int kG, bool kAll, uint32_t kPos = 0x76543210u>
__global__ void __launch_bounds__(kT * kG + 32, 1) optimize_pipe_kernel(
    const __grid_constant__ PipeBatches B, uint64_t en0, uint64_t en1) {
  static_assert(kS % kG == 0, "each consumer group owns every kG-th stage");
  using L = PipeLayout<kT, kS, kCap>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full_bar[kS], empty_bar[kS];
  __shared__ int s_cnt[kG][2][8];
  __shared__ uint16_t s_order[kG][kT];
  __shared__ double s_obj[kG][2][kT];
  __shared__ uint8_t s_cand[kG][2][kT];

  const int tid = threadIdx.x;
  const uint64_t ntiles = B.tile0[B.nb];
  if (tid == 0) TRACE(4095);
  if (tid == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kEmptyArrivals<kT>);
    }
    fence_mbar_init();
  }
  if (tid < kG * 16) (&s_cnt[0][0][0])[tid] = 0;
  // Programmatic dependent launch: the shared-memory prologue above overlaps the previous grid
  // on the stream; let the next grid be scheduled now (its CTAs take over SMs as ours retire),
  // then wait until every earlier grid has completed and its writes are visible before
  // touching global memory. Both are no-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();

  auto stage_base = [&](int s) { return smem + size_t(s) * L::kStageBytes; };

  if (tid >= kT * kG) {
    // ------------------------------ producer warp ------------------------------
    const int lane = tid & 31;
    // lane b: the end of batch b's speed rows (a TMA rounded up to 16 bytes stays inside it)
    const uintptr_t my_end =
        lane < B.nb ? reinterpret_cast<uintptr_t>(B.speeds[lane] +
                                                  size_t(__ldg(B.offsets[lane] + B.n[lane])) * 5)
                    : 0;
    uint32_t pre0 = 0, pre1 = 0;
    int pre_b = 0, cur = 0;  // lane's prefetched tile batch / its batch cursor
    int k = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
      if ((k & 31) == 0) {
        const uint64_t tl = tile + uint64_t(lane) * gridDim.x;
        if (tl < ntiles) {
          cur = batch_of(B, tl, cur);
          const uint64_t nl = B.n[cur];
          const uint64_t t0l = (tl - B.tile0[cur]) * kT;
          const uint64_t cl = nl - t0l < uint64_t(kT) ? nl - t0l : uint64_t(kT);
          pre0 = __ldg(B.offsets[cur] + t0l);
          pre1 = __ldg(B.offsets[cur] + t0l + cl);
          pre_b = cur;
        }
      }
      const uint32_t o0 = __shfl_sync(0xffffffffu, pre0, k & 31);
      const uint32_t oend = __shfl_sync(0xffffffffu, pre1, k & 31);
      const int b = __shfl_sync(0xffffffffu, pre_b, k & 31);
      const uintptr_t speeds_end = __shfl_sync(0xffffffffu, my_end, b);
      const int st = k % kS;
      const uint32_t ph = (k / kS) & 1;
      if (lane == 0) {
        if (k >= kS) mbar_wait(&empty_bar[st], ph ^ 1);
        TRACE(k * 16 + 3);
        const double* speeds = B.speeds[b];
        const uint32_t* offsets = B.offsets[b];
        const uint64_t n = B.n[b];
        const uint64_t t0 = (tile - B.tile0[b]) * kT;
        const uint32_t cnt = static_cast<uint32_t>(n - t0 < uint64_t(kT) ? n - t0 : uint64_t(kT));
        unsigned char* base = stage_base(st);
        uint32_t* so = reinterpret_cast<uint32_t*>(base);
        // offsets[t0 .. t0+cnt] by whole 16-byte chunks; words of a chunk that would run past
        // offsets[n] (end of the array) are loaded directly instead.
        uint32_t owords = (cnt + 1 + 3) & ~3u;
        uint32_t odirect = 0;
        if (t0 + owords > n + 1) {
          owords = (cnt + 1) & ~3u;
          odirect = cnt + 1 - owords;
        }
        const uint32_t njobs = oend - o0;
        const bool staged = oend >= o0 && njobs <= uint32_t(kCap) && njobs > 0;
        uint32_t rbytes = 0;
        uintptr_t abase = 0, end = 0, aend_tma = 0;
        if (staged) {
          const uintptr_t a0 = reinterpret_cast<uintptr_t>(speeds + size_t(o0) * 5);
          end = a0 + size_t(njobs) * 40;
          abase = a0 & ~uintptr_t(15);
          // Round the end up to 16 bytes when that stays inside the speeds array (the extra
          // <= 8 bytes are the next tile's); otherwise load the trailing double directly.
          const uintptr_t up = (end + 15) & ~uintptr_t(15);
          aend_tma = up <= speeds_end ? up : (end & ~uintptr_t(15));
          rbytes = static_cast<uint32_t>(aend_tma - abase);
        }
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                         smem_u32(&full_bar[st])),
                     "r"(owords * 4 + rbytes)
                     : "memory");
        if (owords) bulk_g2s(so, offsets + t0, owords * 4, &full_bar[st]);
        unsigned char* rows = base + L::kOffWords * 4;
        if (rbytes) bulk_g2s(rows, reinterpret_cast<const void*>(abase), rbytes, &full_bar[st]);
        for (uint32_t w = 0; w < odirect; ++w) so[owords + w] = __ldg(offsets + t0 + owords + w);
        if (staged && aend_tma < end)
          *reinterpret_cast<double*>(rows + rbytes) =
              __ldg(reinterpret_cast<const double*>(aend_tma));
        mbar_arrive(&full_bar[st]);
      }
      __syncwarp();
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  const int g = tid / kT;   // consumer group
  const int ct = tid % kT;  // thread within group
  const int lane = tid & 31;
  int k = 0;  // this group's tile count; it owns CTA tile numbers kk = g, g+kG, ...
  int b = 0;  // batch cursor
  uint64_t prev_t0 = 0;
  int prev_cnt = 0;
  uint8_t* prev_cand = nullptr;
  double* prev_obj = nullptr;
  for (uint64_t tile = blockIdx.x + uint64_t(g) * gridDim.x; tile < ntiles;
       tile += uint64_t(kG) * gridDim.x) {
    const int kk = k * kG + g;
    ++k;
    const int st = kk % kS;
    const uint32_t ph = (kk / kS) & 1;
    const int p = k & 1;
    b = batch_of(B, tile, b);
    const double* speeds = B.speeds[b];
    const uint64_t n = B.n[b];
    mbar_wait(&full_bar[st], ph);
    if (ct == 0) TRACE(kk * 16 + 6);
    const unsigned char* base = stage_base(st);
    const uint32_t* so = reinterpret_cast<const uint32_t*>(base);
    const uint64_t t0 = (tile - B.tile0[b]) * kT;
    const int cnt = static_cast<int>(n - t0 < uint64_t(kT) ? n - t0 : uint64_t(kT));
    const uint32_t j0 = so[0], oend = so[cnt];
    const uint32_t njobs = oend - j0;
    const bool staged = oend >= j0 && njobs <= uint32_t(kCap) && njobs > 0;  // == producer's
    const uint32_t lead =
        static_cast<uint32_t>(reinterpret_cast<uintptr_t>(speeds + size_t(j0) * 5) & 15);
    const double* srows = reinterpret_cast<const double*>(base + L::kOffWords * 4 + lead);

    int my_m = 0, my_rank = 0;
    if (ct < cnt) {
      my_m = valid_m(so[ct + 1] - so[ct]);
      my_rank = atomicAdd(&s_cnt[g][p][my_m], 1);
    }
    named_bar_sync(1 + g, kT);
    // Everyone finished the previous tile: flush its decisions (coalesced) from buffer p^1.
    if (ct < prev_cnt) {
      prev_cand[prev_t0 + ct] = s_cand[g][p ^ 1][ct];
      prev_obj[prev_t0 + ct] = s_obj[g][p ^ 1][ct];
    }
    if (ct == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s_cnt[g][p ^ 1][q] = 0;
    }
    if (ct < cnt) {
      int bb = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        bb += ((kPos >> (4 * q)) & 15) < ((kPos >> (4 * my_m)) & 15) ? s_cnt[g][p][q] : 0;
      s_order[g][bb + my_rank] = static_cast<uint16_t>(ct);
    }
    named_bar_sync(1 + g, kT);
    if (ct < cnt) {
      const int l = s_order[g][ct];
      const uint32_t o = so[l];
      const int m = valid_m(so[l + 1] - o);
      double obj = 0.0;
      uint8_t c;
      if (staged && o >= j0 && o - j0 + uint32_t(m) <= njobs)
        c = search_any<kAll>(srows + size_t(o - j0) * 5, m, en0, en1, &obj);
      else
        c = search_any<kAll>(speeds + size_t(o) * 5, m, en0, en1, &obj);
      s_cand[g][p][l] = c;
      s_obj[g][p][l] = obj;
    }
    __syncwarp();
#if MISO_SEARCH_ALL_ARRIVE
    mbar_arrive(&empty_bar[st]);  // every consumer thread releases its own reads
#else
    if (lane == 0) mbar_arrive(&empty_bar[st]);  // the warp's reads, ordered by __syncwarp
#endif
    if (ct == 0) TRACE(kk * 16 + 7);
    prev_t0 = t0;
    prev_cnt = cnt;
    prev_cand = B.cand[b];
    prev_obj = B.obj[b];
  }
  named_bar_sync(1 + g, kT);
  if (ct < prev_cnt) {
    const int p = k & 1;
    prev_cand[prev_t0 + ct] = s_cand[g][p][ct];
    prev_obj[prev_t0 + ct] = s_obj[g][p][ct];
  }
}

template <int kT, int kS, int kCap, int kG, bool kAll, uint32_t kPos = 0x76543210u>
cudaError_t launch_pipe_cfg(const SearchBatch* batches, int nb, uint64_t en0, uint64_t en1,
                            cudaStream_t stream) {
  using L = PipeLayout<kT, kS, kCap>;
  auto kern = optimize_pipe_kernel<kT, kS, kCap, kG, kAll, kPos>;
  static int grid_cap = 0;
  if (!grid_cap) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(L::kBytes));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT * kG + 32, L::kBytes);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  PipeBatches B;
  B.nb = nb;
  B.tile0[0] = 0;
  for (int i = 0; i < nb; ++i) {
    B.speeds[i] = batches[i].speeds;
    B.offsets[i] = batches[i].offsets;
    B.cand[i] = batches[i].cand;
    B.obj[i] = batches[i].obj;
    B.n[i] = batches[i].n;
    B.tile0[i + 1] = B.tile0[i] + (batches[i].n + kT - 1) / kT;
  }
  for (int i = nb; i < kMaxPipeBatches; ++i) {
    B.speeds[i] = nullptr;
    B.offsets[i] = nullptr;
    B.cand[i] = nullptr;
    B.obj[i] = nullptr;
    B.n[i] = 0;
    B.tile0[i + 1] = B.tile0[nb];
  }
  const uint64_t tiles = B.tile0[nb];
  if (tiles == 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(tiles < uint64_t(grid_cap) ? tiles : uint64_t(grid_cap));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kT * kG + 32);
  cfg.dynamicSmemBytes = L::kBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = use_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, B, en0, en1);
}

// MISO_B200_PIPE_CFG selects a tile/stage/group configuration (tuning only).
static int pipe_cfg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MISO_B200_PIPE_CFG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <bool kAll>
cudaError_t launch_pipe(const SearchBatch* bs, int nb, uint64_t en0, uint64_t en1,
                        cudaStream_t stream) {
  switch (pipe_cfg()) {
    case 1: return launch_pipe_cfg<128, 8, 640, 4, kAll>(bs, nb, en0, en1, stream);
    case 2: return launch_pipe_cfg<128, 6, 640, 3, kAll>(bs, nb, en0, en1, stream);
    case 3: return launch_pipe_cfg<256, 4, 1280, 2, kAll>(bs, nb, en0, en1, stream);
    // bucket order 3,2,5,7,6,1,4 (bad m last): adjacent buckets pair cheap and expensive
    // searches (max adjacent cost 268 vs 361 for ascending m; costs ~ candidates + loads)
    default: return launch_pipe_cfg<256, 4, 1280, 2, kAll, 0x34260157u>(bs, nb, en0, en1, stream);
  }
}

template <bool kAll>
cudaError_t launch_tile(const double* speeds, const uint32_t* offsets, uint64_t n, uint8_t* cand,
                        double* obj, uint64_t en0, uint64_t en1, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(optimize_tile_kernel<kAll>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kTileStageBytes));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const uint64_t blocks = (n + kTile - 1) / kTile;
  optimize_tile_kernel<kAll><<<static_cast<unsigned>(blocks), kTile, kTileStageBytes, stream>>>(
      speeds, offsets, n, cand, obj, en0, en1);
  return cudaGetLastError();
}

constexpr uint64_t kAllEn0 = ~0ull, kAllEn1 = (1ull << (kNumCands - 64)) - 1;

cudaError_t launch_optimize_batches(const SearchBatch* batches, int nb, uint64_t en0,
                                    uint64_t en1, cudaStream_t stream) {
  const bool all = en0 == kAllEn0 && en1 == kAllEn1;
  // 16-byte aligned batches go through the TMA pipeline, up to kMaxPipeBatches per launch;
  // the rest (or MISO_B200_SIMPLE_SEARCH=1) through the one-shot tile kernel.
  SearchBatch piped[kMaxPipeBatches];
  int np = 0;
  auto flush = [&]() -> cudaError_t {
    cudaError_t e = np ? (all ? launch_pipe<true>(piped, np, en0, en1, stream)
                              : launch_pipe<false>(piped, np, en0, en1, stream))
                       : cudaSuccess;
    np = 0;
    return e;
  };
  for (int i = 0; i < nb; ++i) {
    const SearchBatch& bt = batches[i];
    if (bt.n == 0) continue;
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(bt.speeds) | reinterpret_cast<uintptr_t>(bt.offsets)) & 15) == 0;
    if (aligned && !force_simple_path()) {
      piped[np++] = bt;
      if (np == kMaxPipeBatches)
        if (cudaError_t e = flush()) return e;
      continue;
    }
    cudaError_t e = all ? launch_tile<true>(bt.speeds, bt.offsets, bt.n, bt.cand, bt.obj, en0, en1, stream)
                        : launch_tile<false>(bt.speeds, bt.offsets, bt.n, bt.cand, bt.obj, en0, en1, stream);
    if (e) return e;
  }
  return flush();
}

cudaError_t launch_optimize(const double* speeds, const uint32_t* offsets, uint64_t n,
                            uint8_t* cand, double* obj, uint64_t en0, uint64_t en1,
                            cudaStream_t stream) {
  const SearchBatch b{speeds, offsets, n, cand, obj};
  return launch_optimize_batches(&b, 1, en0, en1, stream);
}

}  // namespace miso_b200

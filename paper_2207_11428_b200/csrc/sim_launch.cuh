// sim_launch.cuh -- the simulator kernel and its launcher, included only by the per-policy TUs
// (sim_pol_*.cu), each of which explicitly instantiates its policy.
#pragma once
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "sim_engine.cuh"

// Resident one-warp blocks per SM: the dynamic policies (miso, oracle) carry the predictor and
// the partition search and get 112 registers without spills at 16 per SM; nopart/optsta fit
// 64 registers at 32 per SM (the best-static search runs ~17 candidates per trace).
#ifndef MISO_SIM_MIN_BLOCKS_DYN
#define MISO_SIM_MIN_BLOCKS_DYN 16
#endif
#ifndef MISO_SIM_MIN_BLOCKS
#define MISO_SIM_MIN_BLOCKS 32
#endif
// ASYNC (engine warp + STP helper warp per block): 8 two-warp blocks per SM keep the engine's
// register budget of the one-warp dynamic kernels
#ifndef MISO_SIM_MIN_BLOCKS_ASYNC
#define MISO_SIM_MIN_BLOCKS_ASYNC 8
#endif

namespace miso_b200 {

template <int POL, bool PRUNE, bool LOG, bool STP, bool ASYNC>
__global__ void __launch_bounds__(ASYNC ? 64 : 32,
                                  ASYNC ? MISO_SIM_MIN_BLOCKS_ASYNC
                                        : ((POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE)
                                               ? MISO_SIM_MIN_BLOCKS_DYN : MISO_SIM_MIN_BLOCKS))
simulate_kernel(SimBatch b, SimParams prm, ModelW w) {
  using E = simk::Engine<POL, PRUNE, LOG, STP, ASYNC>;
  if constexpr (ASYNC) {
    if (static_cast<int>(blockIdx.x) >= b.n_seeds) return;
    if (threadIdx.x >= 32) {  // warp 1: the STP helper
      E::stp_helper_main();
      return;
    }
  }
  E::run(b, prm, w);
}

// The engine uses ~2.5 KB of shared memory per block and lives on L1 hits (job records, event
// slots, dense per-job arrays): the unified L1/shared array is split so that shared memory
// holds exactly the resident blocks' records and the rest is L1.
// MISO_B200_SIM_CARVEOUT=<percent shared> overrides it (-1 = the driver's default choice).
inline int sim_carveout_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("MISO_B200_SIM_CARVEOUT");
    v = e ? atoi(e) : -3;  // -3: computed per kernel
  }
  return v;
}

// SMs the launch stream's kernels can use: the device's, or its green context's SM partition
// (driver entry points looked up at run time, so the library links no libcuda).
inline int sim_stream_sms(cudaStream_t stream) {
  static int dev_sms = 0;
  if (dev_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev_sms <= 0) dev_sms = 148;
  }
  using GetGreen = CUresult (*)(CUstream, CUgreenCtx*);
  using GetRes = CUresult (*)(CUgreenCtx, CUdevResource*, CUdevResourceType);
  static GetGreen get_green = nullptr;
  static GetRes get_res = nullptr;
  static bool looked = false;
  if (!looked) {
    looked = true;
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamGetGreenCtx", &f1, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuGreenCtxGetDevResource", &f2, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      get_green = reinterpret_cast<GetGreen>(f1);
      get_res = reinterpret_cast<GetRes>(f2);
    }
  }
  if (get_green && stream) {
    CUgreenCtx g = nullptr;
    CUdevResource r{};
    if (get_green(static_cast<CUstream>(stream), &g) == CUDA_SUCCESS && g &&
        get_res(g, &r, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS && r.sm.smCount > 0)
      return static_cast<int>(r.sm.smCount);
  }
  return dev_sms;
}

// The asynchronous-STP variant (an STP helper warp beside each engine warp) for the dynamic
// policies when the tasks fit the SMs the launch stream can use in about one wave -- a
// latency-bound batch, where taking the STP chain off the engine's critical path pays; a
// many-wave batch keeps one-warp blocks (twice the resident tasks). MISO_B200_SIM_ASYNC_STP=0/1
// forces it off/on.
inline bool sim_async_stp(int n_tasks, cudaStream_t stream) {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("MISO_B200_SIM_ASYNC_STP");
    mode = e ? atoi(e) : -1;
  }
  if (mode >= 0) return mode != 0;
  return n_tasks <= sim_stream_sms(stream) * MISO_SIM_MIN_BLOCKS_ASYNC;
}

template <int POL, bool PRUNE, bool LOG, bool STP, bool ASYNC = false>
cudaError_t launch_sim_k(const SimBatch& b, const SimParams& p, const ModelW& w, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    attr_set = true;
    auto kern = simulate_kernel<POL, PRUNE, LOG, STP, ASYNC>;
    int pct = sim_carveout_env();
    if (pct == -3) {
      cudaFuncAttributes fa{};
      int dev = 0, smem_sm = 0, blocks = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
      if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && smem_sm > 0 &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, ASYNC ? 64 : 32, 0) == cudaSuccess) {
        const size_t need = size_t(blocks) * (fa.sharedSizeBytes + 1024);  // + per-block reserve
        pct = static_cast<int>(std::min<size_t>(100, (need * 100 + smem_sm - 1) / smem_sm));
      } else {
        pct = -1;
      }
    }
    if (pct >= 0) {
      const cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (e != cudaSuccess) return e;
    }
  }
  // one block per task: the engine warp (and with ASYNC the STP helper warp)
  simulate_kernel<POL, PRUNE, LOG, STP, ASYNC><<<b.n_seeds, ASYNC ? 64 : 32, 0, s>>>(b, p, w);
  return cudaGetLastError();
}

// The event-log variant only when a log is requested (pruned runs never take one); the STP
// variant only when the STP is tracked.
template <int POL, bool PRUNE>
cudaError_t launch_sim(const SimBatch& b, const SimParams& p, const ModelW& w, cudaStream_t s) {
  if constexpr (!PRUNE) {
    if (b.log)
      return p.track_stp ? launch_sim_k<POL, PRUNE, true, true>(b, p, w, s)
                         : launch_sim_k<POL, PRUNE, true, false>(b, p, w, s);
  } else {
    if (b.log) return cudaErrorInvalidValue;
  }
  if constexpr (!PRUNE && (POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE)) {
    if (p.track_stp && sim_async_stp(b.n_seeds, s)) return launch_sim_k<POL, PRUNE, false, true, true>(b, p, w, s);
  }
  return p.track_stp ? launch_sim_k<POL, PRUNE, false, true>(b, p, w, s)
                     : launch_sim_k<POL, PRUNE, false, false>(b, p, w, s);
}

}  // namespace miso_b200

// sim_launch.cuh -- the simulator kernel and its launcher, included only by the per-policy TUs
// (sim_pol_*.cu), each of which explicitly instantiates its policy.
#pragma once
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

namespace miso_b200 {

template <int POL, bool PRUNE>
__global__ void __launch_bounds__(32, (POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE)
                                          ? MISO_SIM_MIN_BLOCKS_DYN : MISO_SIM_MIN_BLOCKS)
simulate_kernel(SimBatch b, SimParams prm, ModelW w) {
  simk::Engine<POL, PRUNE>::run(b, prm, w);
}

template <int POL, bool PRUNE>
cudaError_t launch_sim(const SimBatch& b, const SimParams& p, const ModelW& w, cudaStream_t s) {
  simulate_kernel<POL, PRUNE><<<b.n_seeds, 32, 0, s>>>(b, p, w);  // one warp (block) per task
  return cudaGetLastError();
}

}  // namespace miso_b200

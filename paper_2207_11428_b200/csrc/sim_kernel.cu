// sim_kernel.cu -- kernel (c)'s host side: workspace sizing and the per-policy launch dispatch.
// The engine (sim_engine.cuh) is instantiated once per policy in sim_pol_*.cu.
#include <cuda_runtime.h>

#include <algorithm>

#include "sim_engine.cuh"

namespace miso_b200 {

size_t sim_workspace_stride(int max_jobs, int cluster_size) {
  return sim_ws_total(max_jobs, cluster_size);
}

size_t sim_sizeof_job() { return sizeof(simk::DJob); }
size_t sim_sizeof_gpu() { return sizeof(simk::DGpu); }

namespace {
__global__ void __launch_bounds__(256) sim_draws_kernel(const uint64_t* __restrict__ rng_seed,
                                                        int n_tasks, int k, double* __restrict__ out) {
  const size_t total = size_t(n_tasks) * size_t(k) * 14;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(i & 1), col = static_cast<int>((i >> 1) % 7);
    const size_t rest = i / 14;
    const uint64_t nonce = rest % size_t(k) + 1;
    const size_t task = rest / size_t(k);
    out[i] = pack_draw(column_draw(rng_seed[task], nonce, col, e));
  }
}
}  // namespace

cudaError_t launch_sim_draws(const uint64_t* rng_seed, int n_tasks, int k, double* out,
                             cudaStream_t stream) {
  if (n_tasks <= 0 || k <= 0) return cudaSuccess;
  const size_t total = size_t(n_tasks) * size_t(k) * 14;
  const size_t blocks = std::min<size_t>((total + 255) / 256, size_t(148) * 64);
  sim_draws_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(rng_seed, n_tasks, k, out);
  return cudaGetLastError();
}

cudaError_t launch_simulate(const SimBatch& b, const SimParams& p, const double* w2,
                            const double* w1, cudaStream_t stream) {
  if (b.n_seeds == 0) return cudaSuccess;
  ModelW w;
  for (int i = 0; i < 4; ++i) {
    w.w2[i] = w2[i];
    w.w1[i] = w1[i];
  }
  switch (p.policy) {
    case MISO_B200_POLICY_NOPART: return launch_sim<MISO_B200_POLICY_NOPART, false>(b, p, w, stream);
    case MISO_B200_POLICY_OPTSTA:
      return b.prune_bound ? launch_sim<MISO_B200_POLICY_OPTSTA, true>(b, p, w, stream)
                           : launch_sim<MISO_B200_POLICY_OPTSTA, false>(b, p, w, stream);
    case MISO_B200_POLICY_ORACLE: return launch_sim<MISO_B200_POLICY_ORACLE, false>(b, p, w, stream);
    case MISO_B200_POLICY_MISO: return launch_sim<MISO_B200_POLICY_MISO, false>(b, p, w, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace miso_b200

// sim_kernel_prune.cu -- simulate_kernel built a second time with the pruned best-static
// search's bound bookkeeping (MISO_SIM_PRUNE=1, namespace sim_prune): the chosen-only
// candidate runs of miso_b200_simulate_batch_pruned use this kernel, every other simulation
// the plain one, which carries none of the bookkeeping.
#define MISO_SIM_PRUNE 1
#include "sim_kernel.cu"

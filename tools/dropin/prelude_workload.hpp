// Force-included (-include) before the reference's workload_test.cpp to run it against the
// device trace generator: the reference headers are compiled first (their real definitions),
// then later mentions of generate_trace in the test file resolve to the B200 binding
// (include/miso_b200_experiment.hpp, miso_b200_generate_traces_device_host).
#pragma once
#include "miso/common.hpp"
#include "miso/topology.hpp"
#include "miso/profiles.hpp"
#include "miso/optimizer.hpp"
#include "miso/workload.hpp"
#include "miso/sim.hpp"
#include "miso/experiment.hpp"
#include "miso_b200_experiment.hpp"
namespace miso {
inline JobTrace b200_generate_trace_dropin(const TraceSpec& spec) { return b200::generate_trace(spec); }
}  // namespace miso
#define generate_trace b200_generate_trace_dropin

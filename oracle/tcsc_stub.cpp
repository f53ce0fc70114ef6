// Link stub (TEST INFRASTRUCTURE ONLY). proj/src/pipeline.cpp:222-224 references
// dcsc::solve_coding_tcsc for ChannelMode::Joint with J > 1, which is off the
// hot path (every BASELINE config is J = 1) and needs Eigen3, absent here.
#include <stdexcept>

#include "dcsc/tcsc.hpp"

namespace dcsc {

SparseMaps solve_coding_tcsc(const SignalTensor&, const Dictionary&, const SolverConfig&,
                             CodingDualState&, CodingStats*, BlockSolveMethod) {
  throw DimensionError("oracle build: the TCSC (J > 1) path is not compiled (needs Eigen3)");
}

}  // namespace dcsc
